"""Attention-site LUT GEMMs on the tcgen05 kernel.

q | k | v run as one launch on one A4 quantization (model.py:353-358 with the
_site_value cache); each site matches the CPU oracle's LUT GEMM on the same
codes, and the stacked launch is bitwise equal to separate launches."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import oracle as o  # noqa: E402
from paper_2604_10496_b200 import ShapeError, lut_gemm_tc, quantize_activations  # noqa: E402
from paper_2604_10496_b200.attention import OutLinear, QKVLinear, stack_rows  # noqa: E402
from paper_2604_10496_b200.lutgemm import PackedClusteredWeights  # noqa: E402
from paper_2604_10496_b200.synthetic import round_bf16  # noqa: E402


def _site(rng, d_out, d_in, g, kc=16):
    cent = (rng.standard_normal((d_out, d_in // g, 16)) / np.sqrt(d_in)).astype(np.float32)
    cent[:, :, kc:] = 0.0
    ids = rng.integers(0, kc, (d_out, d_in)).astype(np.uint8)
    packed = (ids[:, 0::2] | (ids[:, 1::2] << 4)).astype(np.uint8)
    return cent, packed


@pytest.mark.parametrize("n,d,g,kc", [(1, 512, 128, 16), (37, 1024, 128, 16), (64, 512, 512, 8), (200, 768, 128, 16)])
def test_qkv_one_launch_matches_oracle_and_separate_launches(n, d, g, kc):
    rng = np.random.default_rng(n + d + kc)
    sites = [_site(rng, d, d, g, kc) for _ in range(4)]
    pws = [PackedClusteredWeights(c, i, d, g) for c, i in sites]
    x = round_bf16(rng.standard_normal((n, d)).astype(np.float32))
    qkv = QKVLinear(*pws[:3])
    got = qkv(torch.from_numpy(x).cuda())
    codes, scales = oracle.c_quantize(x)
    for (c, i), out in zip(sites[:3], got):
        want = oracle.c_lut_gemm(codes, scales, i, c, g)
        assert o.relative_error(out.cpu().numpy(), want) <= 2e-6
    qa = quantize_activations(torch.from_numpy(x).cuda())
    for pw, out in zip(pws[:3], got):
        assert torch.equal(lut_gemm_tc(qa, pw, 3, "umma128u"), out)
    # the out projection on its own quantization of the attention output
    attn = round_bf16(rng.standard_normal((n, d)).astype(np.float32))
    proj = OutLinear(pws[3])(torch.from_numpy(attn).cuda())
    ac, asc = oracle.c_quantize(attn)
    assert o.relative_error(proj.cpu().numpy(), oracle.c_lut_gemm(ac, asc, sites[3][1], sites[3][0], g)) <= 2e-6


def test_stack_rows_checks_shapes():
    rng = np.random.default_rng(1)
    a = PackedClusteredWeights(*_site(rng, 128, 256, 128), 256, 128)
    b = PackedClusteredWeights(*_site(rng, 128, 512, 128), 512, 128)
    with pytest.raises(ShapeError):
        stack_rows((a, b))
