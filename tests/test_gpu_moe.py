"""GPU parity of the MoE-layer operator against the composed reference path.

Bit-exact: layer-input codes and scales, router logits, selected experts and
their order, segment offsets and the permutation.  ulp-bounded: route weights
(CUDA expf vs numpy float32 exp).  Tolerance (BASELINE north star): layer
output Frobenius relative error <= 1e-2 vs the reference fp32 LUT path; the
fp32 and ordered device paths are expected near 1e-6."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import oracle as o  # noqa: E402
from paper_2604_10496_b200 import MoELayer  # noqa: E402
from paper_2604_10496_b200.synthetic import (input_digest, moe_inputs_device,  # noqa: E402
                                             moe_inputs_host, to_device_experts)
from paper_2604_10496_b200.moe import ExpertStack  # noqa: E402
from paper_2604_10496_b200 import _lib  # noqa: E402

LAYER_TOL = 1e-2


def _layer(g, path):
    seed, n, d, ff, E, k, gs = (int(v) for v in g["config"])
    v, w, experts, _ = moe_inputs_host(seed, n, d, ff, E, gs)
    assert input_digest(v, w, experts) == str(g["digest"])
    return v, MoELayer(w, to_device_experts(experts), k, path=path), k, E


def _check_routing(layer, tr, g, v, k, E):
    assert np.array_equal(tr["codes"].cpu().numpy(), g["codes"])
    assert np.array_equal(tr["scales"].cpu().numpy().view(np.uint32), g["scales"].view(np.uint32))
    assert np.array_equal(tr["logits"].cpu().numpy().view(np.int32), g["logits"].view(np.int32))
    assert np.array_equal(tr["selected"].cpu().numpy(), g["selected"])
    ulp = np.abs(tr["weights"].cpu().numpy().view(np.int32) - g["weights"].astype(np.float32).view(np.int32))
    assert ulp.max() <= 8
    tok, slot, off, inv = o.route_permutation(g["selected"], E)
    assert np.array_equal(tr["offsets"].cpu().numpy(), off)
    R = off[-1]
    assert np.array_equal(tr["perm_token"].cpu().numpy()[:R], tok)
    assert np.array_equal(tr["perm_slot"].cpu().numpy()[:R], slot)
    assert np.array_equal(tr["inv"].cpu().numpy(), inv)
    assert np.array_equal(tr["codes_perm"].cpu().numpy()[:R], g["codes"][tok])


@pytest.mark.parametrize("name", ["moe_small.npz", "moe_odd.npz", "moe_c1.npz"])
@pytest.mark.parametrize("path", ["f32", "ordered"])
def test_moe_layer_golden(golden, name, path):
    g = golden(name)
    v, layer, k, E = _layer(g, path)
    x = torch.from_numpy(v).cuda()
    out = layer(x).cpu().numpy()
    _check_routing(layer, layer.trace(v.shape[0]), g, v, k, E)
    err = o.relative_error(out, g["out"])
    assert err <= (1e-5 if path != "tc" else LAYER_TOL), err
    # bf16 input of the same (bf16-exact) values gives the identical result
    out_b = layer(x.to(torch.bfloat16)).cpu().numpy()
    assert np.array_equal(out_b.view(np.int32), out.view(np.int32))


def test_moe_layer_deterministic_and_graph_capturable(golden):
    g = golden("moe_c1.npz")
    v, layer, k, E = _layer(g, "auto")
    x = torch.from_numpy(v).cuda()
    a = layer(x).clone()
    out = torch.empty_like(a)
    layer(x, out=out)  # warm workspace
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        layer(x, out=out)
    out.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, a)


def test_moe_top_k_equals_experts_and_ties():
    # top_k = E recovers the full softmax order; equal logits break to lower ids
    v, w, experts, _ = moe_inputs_host(5, 12, 64, 64, 4, 32)
    w0 = np.zeros_like(w)
    layer = MoELayer(w0, to_device_experts(experts), 4, path="f32")
    out = layer(torch.from_numpy(v).cuda()).cpu().numpy()
    tr = layer.trace(12)
    assert np.array_equal(tr["selected"].cpu().numpy(), np.tile(np.arange(4), (12, 1)))
    assert np.allclose(tr["weights"].cpu().numpy(), 0.25)
    want = oracle.moe_layer_fast(v, w0, experts, 4)
    assert o.relative_error(out, want) <= 1e-5


def test_mixtral_decode_vs_oracle_subsample_and_ordered():
    """Mixtral-8x7B layer shape (d=4096, ff=14336, E=8, top-2), decode b=64."""
    n, d, ff, E, k, g = 64, 4096, 14336, 8, 2, 128
    v, w, sites, _ = moe_inputs_device(11, n, d, ff, E, g)
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, path="f32")
    out = layer(v).float()
    tr = {k_: t.clone() for k_, t in layer.trace(n).items()}
    ordered = layer(v, path="ordered").float()
    tro = layer.trace(n, path="ordered")
    # identical routing / permutation / codes on both paths
    for key in ("codes", "scales", "logits", "selected", "offsets", "perm_token", "inv"):
        assert torch.equal(tr[key], tro[key]), key
    R = int(tr["offsets"][-1])
    # the gate|up GEMMs agree to fp32 accumulation-order noise on identical codes
    assert o.relative_error(tr["hidden"][:R].cpu().numpy(), tro["hidden"][:R].cpu().numpy()) <= 1e-5
    # the layer output differs only through isolated 4-bit re-quantization flips
    assert o.relative_error(out.cpu().numpy(), ordered.cpu().numpy()) <= LAYER_TOL
    # CPU oracle on a token subsample (routing and quantization are per token)
    sub = 6
    host_experts = []
    for e in range(E):
        mats = []
        for s in ("gate", "up", "down"):
            ids, cents, di, do = sites[s]
            mats.append((cents[e].cpu().numpy(), ids[e].cpu().numpy(), g))
        host_experts.append(mats)
    want = oracle.moe_layer_fast(v[:sub].float().cpu().numpy(), w.cpu().numpy(), host_experts, k)
    assert o.relative_error(ordered[:sub].cpu().numpy(), want) <= LAYER_TOL
    assert o.relative_error(out[:sub].cpu().numpy(), want) <= LAYER_TOL


def _host_experts(sites, n_exp, g):
    out = []
    for e in range(n_exp):
        out.append([(sites[s][1][e].cpu().numpy(), sites[s][0][e].cpu().numpy(), g) for s in ("gate", "up", "down")])
    return out


@pytest.mark.parametrize("E,k,n", [(32, 6, 300), (64, 6, 300), (128, 8, 300), (16, 2, 300), (128, 8, 4100),
                                   (64, 6, 8200), (16, 2, 4100)])
def test_router_many_experts_bit_exact(E, k, n):
    """Routing at the QW / DS / PH expert counts (the register-tiled router
    kernel for E in {32, 64, 128}; 16-token tiles at n = 300, 4096 / E-token
    tiles with a ragged last one at n * E >= 128 * 4096): logits and the selected
    experts bit-exact with the ordered chain of _core.matmul_f32 +
    select_top_k; weights ulp-bounded."""
    d, ff, g = 1024, 128, 128
    v, w, sites, _ = moe_inputs_device(23 + E, n, d, ff, E, g)
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, path="f32")
    layer(v)
    tr = layer.trace(n)
    vh = v.float().cpu().numpy()
    codes, scales = oracle.c_quantize(vh)
    logits = oracle.c_matmul(codes.astype(np.float32) * scales[:, None], w.cpu().numpy())
    sel, wts = o.select_top_k(logits, k)
    assert np.array_equal(tr["logits"].cpu().numpy().view(np.int32), logits.view(np.int32))
    assert np.array_equal(tr["selected"].cpu().numpy(), sel)
    ulp = np.abs(tr["weights"].cpu().numpy().view(np.int32) - wts.astype(np.float32).view(np.int32))
    assert ulp.max() <= 8
    tok, slot, off, inv = o.route_permutation(sel, E)
    assert np.array_equal(tr["offsets"].cpu().numpy(), off)
    assert np.array_equal(tr["inv"].cpu().numpy(), inv)


@pytest.mark.parametrize("n,d,E", [(1, 1024, 8), (64, 4096, 8), (130, 1040, 8), (296, 1024, 8), (7, 2048, 16),
                                   (200, 1024, 16), (64, 2048, 64), (33, 1024, 128), (5, 1040, 24), (64, 1024, 32)])
def test_router_decode_chain_bit_exact(n, d, E):
    """Decode-sized batches take router_chain_kernel (chains alone on warp 0,
    products from warps 1-3): logits bit-exact with _core.matmul_f32's ordered
    chain, for 8/16/32-expert groups, several tokens per CTA and a partial
    last chunk (d = 1040)."""
    g = 16
    v, w, sites, _ = moe_inputs_device(50 + n + E, n, d, 128, E, g)
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=2, path="f32")
    layer(v)
    tr = layer.trace(n)
    codes, scales = oracle.c_quantize(v.float().cpu().numpy())
    logits = oracle.c_matmul(codes.astype(np.float32) * scales[:, None], w.cpu().numpy())
    assert np.array_equal(tr["logits"].cpu().numpy().view(np.int32), logits.view(np.int32))
    sel, wts = o.select_top_k(logits, 2)
    assert np.array_equal(tr["selected"].cpu().numpy(), sel)
    # E <= 32: the same launch did top-k and the permutation (last CTA); E > 32: separate kernels
    ulp = np.abs(tr["weights"].cpu().numpy().view(np.int32) - wts.astype(np.float32).view(np.int32))
    assert ulp.max() <= 8
    tok, slot, off, inv = o.route_permutation(sel, E)
    R = int(off[-1])
    assert np.array_equal(tr["offsets"].cpu().numpy(), off)
    assert np.array_equal(tr["perm_token"].cpu().numpy()[:R], tok)
    assert np.array_equal(tr["perm_slot"].cpu().numpy()[:R], slot)
    assert np.array_equal(tr["inv"].cpu().numpy(), inv)
    # a second call starts from cleared counts (the quantizer zeroes them)
    layer(v)
    assert np.array_equal(layer.trace(n)["offsets"].cpu().numpy(), off)


@pytest.mark.parametrize("n,E,k", [(1, 8, 2), (64, 8, 2), (33, 16, 4), (100, 32, 8), (296, 8, 2), (7, 24, 3),
                                   (64, 128, 8), (100, 64, 6), (1, 128, 8), (200, 128, 8)])
def test_tc_decode_route_mode(n, E, k):
    """Tensor-core forward at decode sizes: the router launch also does top-k
    (one expert group) or the GEMM's B build takes it from the logits (E > 32,
    n <= 128), and the B build derives the segment permutation in every CTA
    (route_perm.cuh) and publishes it; n = 200 at E = 128 runs the separate
    kernels.  With one expert group the router launch quantizes too (fp32 and
    bf16 inputs).  Routing arrays bit-exact with the
    oracle, the layer output within the layer tolerance of the ordered path,
    and identical across two calls."""
    d, ff, g = 256, 256, 128
    v, w, sites, _ = moe_inputs_device(90 + n + E, n, d, ff, E, g)
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, path="tc")
    layer.prepare_tc()
    out = layer(v).clone()
    tr = layer.trace(n)
    codes, scales = oracle.c_quantize(v.float().cpu().numpy())
    logits = oracle.c_matmul(codes.astype(np.float32) * scales[:, None], w.cpu().numpy())
    sel, wts = o.select_top_k(logits, k)
    assert np.array_equal(tr["logits"].cpu().numpy().view(np.int32), logits.view(np.int32))
    assert np.array_equal(tr["selected"].cpu().numpy(), sel)
    ulp = np.abs(tr["weights"].cpu().numpy().view(np.int32) - wts.astype(np.float32).view(np.int32))
    assert ulp.max() <= 8
    tok, slot, off, inv = o.route_permutation(sel, E)
    R = int(off[-1])
    assert np.array_equal(tr["offsets"].cpu().numpy(), off)
    assert np.array_equal(tr["counts"].cpu().numpy()[:E], np.diff(off))
    assert np.array_equal(tr["perm_token"].cpu().numpy()[:R], tok)
    assert np.array_equal(tr["perm_slot"].cpu().numpy()[:R], slot)
    assert np.array_equal(tr["inv"].cpu().numpy(), inv)
    assert np.array_equal(tr["scales_perm"].cpu().numpy()[:R].view(np.int32), scales[tok].view(np.int32))
    # the layer-input codes, scales and code sums (decode: quantized inside the router launch)
    assert np.array_equal(tr["codes"].cpu().numpy(), codes)
    assert np.array_equal(tr["scales"].cpu().numpy().view(np.int32), scales.view(np.int32))
    assert np.array_equal(tr["tok_sums"].cpu().numpy(), codes.astype(np.int32).sum(axis=1))
    ordered = layer(v, path="ordered")
    assert o.relative_error(out.cpu().numpy(), ordered.cpu().numpy()) <= LAYER_TOL
    assert torch.equal(layer(v), out)
    # bf16 input: the same quantizer on the bf16 values, bit for bit
    vb = v.to(torch.bfloat16)
    layer(vb)
    trb = layer.trace(n)
    cb, sb = oracle.c_quantize(vb.float().cpu().numpy())
    assert np.array_equal(trb["codes"].cpu().numpy(), cb)
    assert np.array_equal(trb["scales"].cpu().numpy().view(np.int32), sb.view(np.int32))
    lb = oracle.c_matmul(cb.astype(np.float32) * sb[:, None], w.cpu().numpy())
    assert np.array_equal(trb["logits"].cpu().numpy().view(np.int32), lb.view(np.int32))
    assert np.array_equal(trb["selected"].cpu().numpy(), o.select_top_k(lb, k)[0])


@pytest.mark.parametrize("g", [0, 128])
@pytest.mark.parametrize("outliers", [False, True])
def test_tc_layer_embedding_wise_and_outliers_vs_oracle(g, outliers):
    """SURVEY §8(d)'s second group-size row (g = d_in, one centroid set per
    output row) and the planted-outlier activations (8x channels, 50x rows):
    the tensor-core layer against the composed CPU oracle."""
    n, d, ff, E, k = 48, 256, 384, 8, 2
    v, w, experts, _ = moe_inputs_host(13, n, d, ff, E, g, outliers=outliers)
    if g == 0:
        assert [m[2] for m in experts[0]] == [d, d, ff]
    layer = MoELayer(w, to_device_experts(experts), k, path="tc")
    layer.prepare_tc()
    out = layer(torch.from_numpy(v).cuda()).cpu().numpy()
    want = oracle.moe_layer_fast(v, w, experts, k)
    assert o.relative_error(out, want) <= LAYER_TOL
    ordered = layer(torch.from_numpy(v).cuda(), path="ordered").cpu().numpy()
    assert o.relative_error(ordered, want) <= 1e-5


@pytest.mark.parametrize("n,ff", [(4, 14336), (60, 14336), (140, 14336), (300, 768), (130, 1408), (50, 256),
                                  (40, 6400)])
def test_silu_requant_rows(n, ff):
    """The silu|re-quantize kernels: long rows (ff = 14336) at decode row counts
    take the cluster kernel (8 / 4 / 2 CTAs per row, row max through DSMEM),
    others a CTA per row (one float4 per thread for short rows).  Codes and
    scales are bit-exact with the oracle quantizer on the kernel's own h,
    h = silu(a)*b agrees with the ordered path, and the layer output does not
    depend on keeping h (CQ_FLAG_KEEP_HIDDEN)."""
    d, E, k, g = 256, 4, 2, 128
    v, w, sites, _ = moe_inputs_device(70 + n, n, d, ff, E, g)
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, path="tc")
    layer.prepare_tc()
    plain = layer(v).clone()
    layer.keep_hidden = True  # trace h on the tensor-core path
    assert torch.equal(layer(v), plain)
    tr = {key: t.clone() for key, t in layer.trace(n).items()}
    layer(v, path="ordered")
    tro = layer.trace(n, path="ordered")
    R = n * k
    h = tr["hidden"][:R].cpu().numpy()
    codes, scales = oracle.c_quantize(h)
    assert np.array_equal(tr["hcodes"][:R].cpu().numpy(), codes)
    assert np.array_equal(tr["hscales"][:R].cpu().numpy().view(np.int32), scales.view(np.int32))
    assert o.relative_error(h, tro["hidden"][:R].cpu().numpy()) <= 1e-5


@pytest.mark.parametrize("cfg", ["qw", "ds"])
def test_many_expert_layers_tc_vs_oracle(cfg):
    """QW (d2048/ff768/E128/top-8) and DS (d2048/ff1408/E64+2 shared/top-6)
    layer shapes on the tensor-core path vs the composed CPU oracle."""
    d, ff, E, k, n_sh = {"qw": (2048, 768, 128, 8, 0), "ds": (2048, 1408, 64, 6, 2)}[cfg]
    n, g = 80, 128
    v, w, sites, sh = moe_inputs_device(31, n, d, ff, E, g, n_shared=n_sh)
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    shared = (tuple(ExpertStack(sh[s][0], sh[s][1], sh[s][2], sh[s][3], g) for s in ("gate", "up", "down"))
              if n_sh else None)
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, shared=shared, path="tc")
    layer.prepare_tc()
    out = layer(v).cpu().numpy()
    ordered = layer(v, path="ordered").cpu().numpy()
    want = oracle.moe_layer_fast(v.float().cpu().numpy(), w.cpu().numpy(), _host_experts(sites, E, g), k,
                                 shared=_host_experts(sh, n_sh, g) if n_sh else ())
    assert o.relative_error(ordered, want) <= 1e-6
    assert o.relative_error(out, want) <= LAYER_TOL


@pytest.mark.parametrize("n", [1, 80, 300])
def test_shared_experts_merged_segments(n, monkeypatch):
    """DS-shaped layer: the shared experts as extra segments of the routed launches
    (CQ_FLAG_SHARED_MERGED) give the same bits as their separate launches."""
    d, ff, E, k, n_sh, g = 2048, 1408, 64, 6, 2, 128
    v, w, sites, sh = moe_inputs_device(41, n, d, ff, E, g, n_shared=n_sh)
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    shared = tuple(ExpertStack(sh[s][0], sh[s][1], sh[s][2], sh[s][3], g) for s in ("gate", "up", "down"))
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, shared=shared, path="tc").prepare_tc()
    assert layer.shared_merged() and layer.desc().flags & _lib.FLAG_SHARED_MERGED
    merged = layer(v).cpu()
    monkeypatch.setenv("CQ_SHARED_MERGE", "0")
    assert not layer.desc().flags & _lib.FLAG_SHARED_MERGED
    separate = layer(v).cpu()
    assert torch.equal(merged, separate)


def test_phi_prefill_rotation_tc_vs_oracle():
    """PH shape (d4096/ff6400/E16/top-2) with the online rotation v = x @ R,
    prefill-sized batch: the tensor-core path vs the oracle on a token subsample."""
    n, d, ff, E, k, g = 256, 4096, 6400, 16, 2, 128
    x, w, sites, _ = moe_inputs_device(37, n, d, ff, E, g)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    R = torch.linalg.qr(torch.randn((d, d), generator=gen, device="cuda"))[0].contiguous()
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, rotation=R, path="tc")
    layer.prepare_tc()
    out = layer(x).cpu().numpy()
    sub = 8
    vr = oracle.c_matmul(x[:sub].float().cpu().numpy(), R.cpu().numpy())
    want = oracle.moe_layer_fast(vr, w.cpu().numpy(), _host_experts(sites, E, g), k)
    assert o.relative_error(out[:sub], want) <= LAYER_TOL


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_tensor_core_rotation_fp32_accuracy(dtype):
    """The online rotation on the tensor cores (bf16 input: x loaded by TMA
    against two bf16 planes of R; fp32 input: three planes of x re-laid out,
    six plane products) matches x @ R at fp32 accuracy: Frobenius relative
    error <= 2e-5 vs an fp64 product (fp32 accumulation-order level)."""
    n, d, ff, E, k, g = 200, 1024, 256, 8, 2, 128
    x, w, sites, _ = moe_inputs_device(41, n, d, ff, E, g)
    x = x.to(dtype)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(9)
    R = torch.linalg.qr(torch.randn((d, d), generator=gen, device="cuda"))[0].contiguous()
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, rotation=R, path="tc")
    layer.prepare_tc()
    layer(x)
    buf, offs = layer.workspace(n)
    buf.fill_(0xFF)  # poison the workspace: every operand the kernels read must be written first
    layer(x)
    from paper_2604_10496_b200 import _lib
    o_rot = offs[_lib.WS_NAMES.index("rotated")]
    got = buf[o_rot:o_rot + n * d * 4].view(torch.float32).view(n, d)
    want = (x.double() @ R.double())
    err = (torch.linalg.norm(got.double() - want) / torch.linalg.norm(want)).item()
    # fp32-level: the split keeps ~24 bits; the residual is the tensor core's fp32 accumulation order
    assert err <= 2e-5, err
    # and the layer's routing equals the fp32 CUDA-core rotation's almost everywhere
    f32 = MoELayer.from_stacks(w, *stacks, top_k=k, rotation=R, path="f32")
    f32(x)
    agree = (f32.trace(n)["selected"] == layer.trace(n)["selected"]).all(dim=1).float().mean().item()
    assert agree >= 0.98, agree


@pytest.mark.parametrize("path", ["tc", "f32", "ordered"])
def test_nonfinite_input_raises_divergence_error(path):
    """A non-finite layer input sets the sticky device flag (no host sync in the
    forward); check_finite reads it and raises DivergenceError naming the site,
    like quant.py:93-94 / model.py:307-309, then clears it."""
    from paper_2604_10496_b200 import DivergenceError
    n, d, ff, E, k, g = 20, 256, 256, 4, 2, 128
    v, w, sites, _ = moe_inputs_device(61, n, d, ff, E, g)
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, path=path)
    if path == "tc":
        layer.prepare_tc()
    layer(v, check_finite=True)  # finite: no error
    bad = v.clone()
    bad[3, 7] = float("nan")
    layer(bad)                    # no sync, no raise
    with pytest.raises(DivergenceError, match="router/gate/up"):
        layer.check_finite(n)
    layer.check_finite(n)         # cleared
    bad[3, 7] = float("inf")
    with pytest.raises(DivergenceError):
        layer(bad, check_finite=True)


@pytest.mark.parametrize("path", ["f32", "ordered"])
def test_nonfinite_hidden_raises_at_down_site(path):
    """An inf centroid makes a gate output non-finite: the down-input
    re-quantization flags it (model.py:397-399 site)."""
    from paper_2604_10496_b200 import DivergenceError
    n, d, ff, E, k, g = 16, 256, 256, 4, 4, 128
    v, w, sites, _ = moe_inputs_device(62, n, d, ff, E, g)
    sites["gate"][1][2, 5, 0, :] = float("inf")  # expert 2, row 5, group 0: every centroid
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, path=path)
    with pytest.raises(DivergenceError, match="down input"):
        layer(v, check_finite=True)
