"""Parity at the BASELINE.json configurations, at bench size, on the path the
bench runs (`path="auto"` after `prepare_tc`: the tcgen05 GEMMs), against the
CPU oracle (the C restatement of the reference's kernels, oracle/cq_oracle.c,
pinned to the reference's own outputs by tests/test_oracle.py).

Per configuration, on ALL tokens of the batch:
  * bit-exact: the A4 codes and scales of the layer input (quant.py:89-100),
    the router logits (ordered chain, linalg.py:66-75 -> _core.pyx:27-38), the
    selected experts and their order (model.py:324-330), the segment offsets
    and permutation (builder-defined);
  * ulp-bounded: route weights (numpy vs CUDA expf);
and on a 64-token subsample (routing and quantization are per token, so the
subsample is exact for its rows): the layer output within the north-star
tolerance, Frobenius relative error <= 1e-2 vs the composed reference path
(pipeline.py:349-355's metric).

PH runs the online rotation v = x @ R (pipeline.py:516).  Its ordered form
(`exact_rotation`, and the "ordered"/"f32" paths) reproduces the reference's
chain bit for bit, so routing stays bit-exact; the tcgen05 rotation (three
bf16 planes of R, fp32 tensor-core accumulation) is not an ordered chain, and
its code / routing disagreement with the oracle is measured and bounded
(DESIGN.md §4b)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import oracle as o  # noqa: E402
from paper_2604_10496_b200 import MoELayer  # noqa: E402
from paper_2604_10496_b200.moe import ExpertStack  # noqa: E402
from paper_2604_10496_b200.synthetic import moe_inputs_device  # noqa: E402

LAYER_TOL = 1e-2
SUB = 64

CONFIGS = {  # BASELINE.json configs[1..4] at the bench's sizes
    "mx": dict(n=64, d=4096, ff=14336, E=8, k=2, n_sh=0),      # Mixtral-8x7B decode b=64
    "ph": dict(n=4096, d=4096, ff=6400, E=16, k=2, n_sh=0),    # Phi-3.5-MoE prefill 4096 + rotation
    "qw": dict(n=4096, d=2048, ff=768, E=128, k=8, n_sh=0),    # Qwen3-30B-A3B prefill 4096
    "ds": dict(n=8192, d=2048, ff=1408, E=64, k=6, n_sh=2),    # DeepSeek-V2-Lite prefill 8192 + 2 shared
}


class _LazyExperts:
    """Host copies of an expert stack, fetched only for experts the oracle uses."""

    def __init__(self, sites, n, g):
        self.sites, self.n, self.g, self.cache = sites, n, g, {}

    def __len__(self):
        return self.n

    def __getitem__(self, e):
        if e not in self.cache:
            self.cache[e] = [(self.sites[s][1][e].cpu().numpy(), self.sites[s][0][e].cpu().numpy(), self.g)
                             for s in ("gate", "up", "down")]
        return self.cache[e]


def _build(cfg, seed, rotation=False):
    c = CONFIGS[cfg]
    g = 128
    x, w, sites, sh = moe_inputs_device(seed, c["n"], c["d"], c["ff"], c["E"], g, n_shared=c["n_sh"])
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    shared = (tuple(ExpertStack(sh[s][0], sh[s][1], sh[s][2], sh[s][3], g) for s in ("gate", "up", "down"))
              if c["n_sh"] else None)
    R = None
    if rotation:
        gen = torch.Generator(device="cuda")
        gen.manual_seed(seed + 1)
        R = torch.linalg.qr(torch.randn((c["d"], c["d"]), generator=gen, device="cuda"))[0].contiguous()
    layer = MoELayer.from_stacks(w, *stacks, top_k=c["k"], shared=shared, rotation=R, path="auto").prepare_tc()
    host = dict(w=w.cpu().numpy(), experts=_LazyExperts(sites, c["E"], g),
                shared=[_LazyExperts(sh, c["n_sh"], g)[s] for s in range(c["n_sh"])] if c["n_sh"] else (),
                R=None if R is None else R.cpu().numpy())
    return c, x, layer, host


def _routing_vs_oracle(tr, v, w, k, E):
    """Bit-exact routing of all tokens against the oracle; returns the oracle's codes/scales/selection."""
    codes, scales = oracle.c_quantize(v)
    assert np.array_equal(tr["codes"].cpu().numpy(), codes)
    assert np.array_equal(tr["scales"].cpu().numpy().view(np.int32), scales.view(np.int32))
    logits = oracle.c_matmul(codes.astype(np.float32) * scales[:, None], w)
    assert np.array_equal(tr["logits"].cpu().numpy().view(np.int32), logits.view(np.int32))
    sel, wts = o.select_top_k(logits, k)
    assert np.array_equal(tr["selected"].cpu().numpy(), sel)
    ulp = np.abs(tr["weights"].cpu().numpy().view(np.int32) - wts.astype(np.float32).view(np.int32))
    assert ulp.max() <= 8
    tok, slot, off, inv = o.route_permutation(sel, E)
    R = int(off[-1])
    assert np.array_equal(tr["offsets"].cpu().numpy(), off)
    assert np.array_equal(tr["perm_token"].cpu().numpy()[:R], tok)
    assert np.array_equal(tr["inv"].cpu().numpy(), inv)
    return codes, scales, sel


def _layer_vs_oracle(out, v, host, k):
    want = oracle.moe_layer_fast(v[:SUB], host["w"], host["experts"], k, shared=host["shared"])
    err = o.relative_error(out[:SUB], want)
    assert err <= LAYER_TOL, err
    return err


@pytest.mark.parametrize("cfg", ["mx", "qw", "ds"])
def test_bench_config_tc_path_vs_oracle(cfg):
    c, x, layer, host = _build(cfg, 101)
    out = layer(x, check_finite=True).cpu().numpy()
    assert layer.tc_shapes_ok() and layer.gate.tc is not None  # "auto" on prepared weights: the tcgen05 path
    tr = layer.trace(c["n"])
    v = x.float().cpu().numpy()
    _routing_vs_oracle(tr, v, host["w"], c["k"], c["E"])
    _layer_vs_oracle(out, v, host, c["k"])
    # deterministic run to run
    assert np.array_equal(layer(x).cpu().numpy().view(np.int32), out.view(np.int32))


def test_mixtral_ordered_path_vs_oracle_all_tokens():
    """The bit-exact GPU path at full Mixtral size: every GEMM is the
    reference's ordered chain, so all 64 tokens agree with the CPU oracle up
    to the ulp-level silu / softmax exp differences."""
    c, x, layer, host = _build("mx", 103)
    out = layer(x, path="ordered").cpu().numpy()
    v = x.float().cpu().numpy()
    _routing_vs_oracle(layer.trace(c["n"], path="ordered"), v, host["w"], c["k"], c["E"])
    want = oracle.moe_layer_fast(v, host["w"], host["experts"], c["k"])
    assert o.relative_error(out, want) <= 1e-5


def test_phi_prefill_exact_rotation_bit_exact_routing():
    """PH 4096 tokens with the online rotation in the reference's ordered
    chain on the tensor-core path (`exact_rotation`): v = x @ R bitwise, so
    codes, logits, top-k and the permutation are bit-exact on all tokens."""
    c, x, layer, host = _build("ph", 107, rotation=True)
    layer.exact_rotation = True
    out = layer(x).cpu().numpy()
    tr = layer.trace(c["n"])
    buf, offs = layer.workspace(c["n"])
    from paper_2604_10496_b200 import _lib
    o_rot = offs[_lib.WS_NAMES.index("rotated")]
    got_v = buf[o_rot:o_rot + c["n"] * c["d"] * 4].view(torch.float32).view(c["n"], c["d"]).cpu().numpy()
    v = oracle.c_matmul(x.float().cpu().numpy(), host["R"])       # pipeline.py:516 in the ordered chain
    assert np.array_equal(got_v.view(np.int32), v.view(np.int32))
    _routing_vs_oracle(tr, v, host["w"], c["k"], c["E"])
    _layer_vs_oracle(out, v, host, c["k"])


def test_phi_prefill_tensor_core_rotation_certified_bit_exact():
    """The bench's PH path: the tcgen05 rotation (three bf16 planes of R, fp32
    tensor-core accumulation) followed by the certified quantizer (rotq.cu),
    which recomputes in the reference's ordered chain every element whose code
    the tensor-core value cannot settle and every candidate for the row max.
    On all 4096 tokens the A4 codes, scales, logits, top-k and permutation are
    bit-exact with the oracle's quantize(x @ R) (pipeline.py:516), the layer
    output equals the bit-exact path's within the tolerance, and the recomputed
    elements are a small fraction of the row (measured rates: DESIGN.md §4b)."""
    c, x, layer, host = _build("ph", 107, rotation=True)
    out = layer(x, check_finite=True).cpu().numpy()
    tr = layer.trace(c["n"])
    recomputed = int(tr["status"][2].item())
    v = oracle.c_matmul(x.float().cpu().numpy(), host["R"])           # the reference's chain
    _routing_vs_oracle(tr, v, host["w"], c["k"], c["E"])
    _layer_vs_oracle(out, v, host, c["k"])
    layer.exact_rotation = True
    exact = layer(x, path="ordered").cpu().numpy()
    err = o.relative_error(out, exact)
    print(f"PH certified rotation: {recomputed} of {c['n'] * c['d']} elements recomputed in the ordered chain "
          f"({recomputed / c['n']:.1f} per token); layer vs the bit-exact path over {c['n']} tokens: {err:.2e}")
    assert err <= LAYER_TOL
    assert 0 < recomputed <= 64 * c["n"]


def test_certified_rotation_wide_band_many_rounds(monkeypatch):
    """A 60x wider recompute band (CQ_ROT_CERT_EPS): hundreds of unsettled
    elements per row, several collect/resolve rounds of the certified
    quantizer; the codes and scales are still the ordered chain's bit for bit."""
    monkeypatch.setenv("CQ_ROT_CERT_EPS", "1e-2")
    c = dict(CONFIGS["ph"])
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    n, d = 40, c["d"]
    x = torch.randn((n, d), generator=gen, device="cuda").to(torch.bfloat16)
    R = torch.linalg.qr(torch.randn((d, d), generator=gen, device="cuda"))[0].contiguous()
    x, w, sites, _ = moe_inputs_device(9, n, d, 512, 4, 128)
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], 128) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=2, rotation=R, path="auto").prepare_tc()
    layer(x)
    tr = layer.trace(n)
    assert int(tr["status"][2].item()) > 3 * 128 * n // 4
    v = oracle.c_matmul(x.float().cpu().numpy(), R.cpu().numpy())
    codes, scales = oracle.c_quantize(v)
    assert np.array_equal(tr["codes"].cpu().numpy(), codes)
    assert np.array_equal(tr["scales"].cpu().numpy().view(np.int32), scales.view(np.int32))
