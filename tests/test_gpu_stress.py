"""Randomized layer shapes on the tensor-core path (tools/stress_parity.py in
small): tokens, experts, top-k, widths, group size (128 or embedding-wise) and
codebook size drawn at random.  For each, the tcgen05 layer against the
ordered path within the layer tolerance, the decode and prefill GEMM
geometries bitwise equal, and a repeated call bitwise equal."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import oracle as o  # noqa: E402
from paper_2604_10496_b200.moe import ExpertStack, MoELayer  # noqa: E402
from paper_2604_10496_b200.synthetic import moe_inputs_device  # noqa: E402


def _case(i):
    rng = np.random.default_rng(9000 + i)
    E = int(rng.choice([4, 8, 16, 24, 32, 64, 128]))
    k = int(rng.integers(1, min(8, E) + 1))
    d = int(rng.choice([256, 512, 1024]))
    ff = int(rng.choice([256, 384, 768]))
    n = int(rng.choice([1, 3, 17, 64, 130, 300]))
    g = int(rng.choice([128, 0]))
    kc = int(rng.choice([16, 8, 4]))
    return n, E, k, d, ff, g, kc


@pytest.mark.parametrize("i", range(8))
def test_random_layer_tc_vs_ordered_and_geometries(monkeypatch, i):
    n, E, k, d, ff, g, kc = _case(i)
    v, w, sites, _ = moe_inputs_device(2000 + i, n, d, ff, E, g, kc=kc)
    st = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *st, top_k=k, path="tc")
    layer.prepare_tc()
    out = layer(v).clone()
    assert torch.equal(layer(v), out)
    monkeypatch.setenv("CQ_UMMA_GEOMETRY", "decode")
    dec = layer(v).clone()
    assert torch.equal(dec, out)
    if n * k >= 64:
        monkeypatch.setenv("CQ_UMMA_GEOMETRY", "prefill")
        assert torch.equal(layer(v), dec)
    monkeypatch.delenv("CQ_UMMA_GEOMETRY")
    ref = layer(v, path="ordered")
    assert o.relative_error(out.cpu().numpy(), ref.cpu().numpy()) <= 1e-2
