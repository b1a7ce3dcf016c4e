"""Tensor-core path: prepared layout invariants and parity.

The digit-plane LUTs are checked by decoding them on the host (unsigned
base-128 digits, biased), the ids re-tiling by inverting it, and the GEMM
against the CPU oracle."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import oracle as o  # noqa: E402
from paper_2604_10496_b200 import MoELayer, QuantizedActivations, lut_gemm_tc  # noqa: E402
from paper_2604_10496_b200.lutgemm import PackedClusteredWeights  # noqa: E402
from paper_2604_10496_b200.moe import ExpertStack  # noqa: E402
from paper_2604_10496_b200.synthetic import moe_inputs_device, moe_inputs_host, to_device_experts  # noqa: E402


def _rand_pw(rng, d_out, d_in, g, scale=1.0):
    cent = (rng.standard_normal((d_out, d_in // g, 16)) * scale).astype(np.float32)
    ids = rng.integers(0, 256, (d_out, d_in // 2)).astype(np.uint8)
    return cent, ids, PackedClusteredWeights(torch.from_numpy(cent), torch.from_numpy(ids), d_in, g)


LAYOUTS = ["umma128u"]


@pytest.mark.parametrize("planes", [2, 3])
def test_digit_plane_luts_decode_to_centroids(planes):
    rng = np.random.default_rng(0)
    rows, tr = 256, 128
    cent, ids, pw = _rand_pw(rng, rows, 512, 128, 0.03)
    cent[3] = 0.0  # an all-zero row gets scale 1 and zero digits
    pw = PackedClusteredWeights(torch.from_numpy(cent), torch.from_numpy(ids), 512, 128)
    pw.prepare_tc(planes, "umma128u")
    lut = pw.tc["lut"].cpu().numpy().astype(np.int64)          # tile-ordered [tile][G][tr][P][16]
    rs = pw.tc["rowscale"].cpu().numpy().astype(np.float64)
    G = 512 // 128
    lut = lut.reshape(rows // tr, G, tr, planes, 16).transpose(0, 2, 1, 3, 4).reshape(rows, G, planes, 16)
    m = np.zeros(lut.shape[:2] + (16,), np.int64)
    # unsigned base-128 digits (sign bits clear, so PRMT(P) | PRMT(Q) is exact), biased
    assert lut.min() >= 0 and lut.max() <= 127
    for p in reversed(range(planes)):
        m = m * 128 + lut[:, :, p, :]
    m -= 1 << (7 * planes - 1)
    rec = m * rs[:, None, None]
    err = np.abs(rec - cent.astype(np.float64)).max(axis=(1, 2))
    assert np.all(err <= rs * 0.5 + 1e-30)
    assert rs[3] == 1.0 and not m[3].any()


def test_retired_layouts_are_rejected():
    from paper_2604_10496_b200 import ConfigError
    rng = np.random.default_rng(1)
    _, _, pw = _rand_pw(rng, 128, 256, 128)
    with pytest.raises(ConfigError):
        pw.prepare_tc(3, "mma16")


def test_umma_ids_are_row_blocks_of_packed_ids():
    rng = np.random.default_rng(2)
    cent, ids, pw = _rand_pw(rng, 256, 384, 128)
    pw.prepare_tc(3, "umma128u")
    got = pw.tc["ids"].cpu().numpy().reshape(2, 3, 4, 128, 16)     # [tile][chunk][kstep][row][16 B]
    want = ids.reshape(2, 128, 3, 4, 16).transpose(0, 2, 3, 1, 4)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n,d_in,d_out,g", [(1, 4096, 1024, 128), (7, 1024, 2816, 128), (16, 4096, 512, 4096),
                                             (33, 2048, 768, 128), (64, 1408, 2048, 128), (100, 512, 256, 256),
                                             (130, 1024, 384, 1024)])
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("planes", [2, 3])
def test_lut_gemm_tc_matches_oracle(n, d_in, d_out, g, planes, layout):
    rng = np.random.default_rng(n + d_in + planes)
    cent, ids, pw = _rand_pw(rng, d_out, d_in, g)
    codes = rng.integers(-8, 8, (n, d_in)).astype(np.int8)
    scales = (0.5 + rng.random(n)).astype(np.float32)
    want = oracle.c_lut_gemm(codes, scales, ids, cent, g)
    qa = QuantizedActivations(torch.from_numpy(codes).cuda(), torch.from_numpy(scales).cuda(), 4)
    got = lut_gemm_tc(qa, pw, planes, layout).cpu().numpy()
    tol = 2e-6 if planes == 3 else 2e-4
    assert o.relative_error(got, want) <= tol


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("name", ["moe_small.npz", "moe_c1.npz"])
def test_moe_layer_tc_golden(golden, name, layout):
    g = golden(name)
    seed, n, d, ff, E, k, gs = (int(v) for v in g["config"])
    v, w, experts, _ = moe_inputs_host(seed, n, d, ff, E, gs)
    layer = MoELayer(w, to_device_experts(experts), k, path="tc")
    if d % 128 or ff % 128 or gs % 128:
        pytest.skip("shape outside the tensor-core envelope")
    layer.prepare_tc(layout=layout)
    out = layer(torch.from_numpy(v).cuda()).cpu().numpy()
    tr = layer.trace(n)
    assert np.array_equal(tr["selected"].cpu().numpy(), g["selected"])
    err = o.relative_error(out, g["out"])
    assert err <= 1e-2, err


@pytest.mark.parametrize("layout", LAYOUTS)
def test_mixtral_decode_tc_vs_ordered(layout):
    n, d, ff, E, k, g = 64, 4096, 14336, 8, 2, 128
    v, w, sites, _ = moe_inputs_device(11, n, d, ff, E, g)
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, path="tc").prepare_tc(layout=layout)
    layer.keep_hidden = True  # trace h on the tensor-core path
    out = layer(v).float()
    tr = {key: t.clone() for key, t in layer.trace(n).items()}
    ordered = layer(v, path="ordered").float()
    tro = layer.trace(n, path="ordered")
    R = int(tr["offsets"][-1])
    # gate|up with 3 digit planes: accumulation-order-level agreement on identical codes
    assert o.relative_error(tr["hidden"][:R].cpu().numpy(), tro["hidden"][:R].cpu().numpy()) <= 1e-5
    assert o.relative_error(out.cpu().numpy(), ordered.cpu().numpy()) <= 1e-2
    # and the tc path is deterministic
    again = layer(v).float()
    assert torch.equal(again, out)


@pytest.mark.parametrize("n,d_in,d_out,g,planes", [(256, 1024, 512, 128, 3), (300, 2048, 768, 128, 2),
                                                   (777, 1024, 1408, 256, 3), (1024, 4096, 256, 128, 3),
                                                   (64, 1024, 512, 128, 3), (96, 2048, 384, 128, 2),
                                                   (128, 4096, 1024, 128, 3)])
def test_prefill_geometry_bitwise_equals_decode(monkeypatch, n, d_in, d_out, g, planes):
    """Long segments take the prefill geometry (128-token passes, 64-column
    chunks).  Both geometries accumulate exact int32 digit products, so the
    result is bitwise that of the 32-token decode geometry, and matches the
    oracle within the digit-plane tolerance."""
    rng = np.random.default_rng(n + d_in + planes)
    cent, ids, pw = _rand_pw(rng, d_out, d_in, g)
    codes = rng.integers(-8, 8, (n, d_in)).astype(np.int8)
    scales = (0.5 + rng.random(n)).astype(np.float32)
    qa = QuantizedActivations(torch.from_numpy(codes).cuda(), torch.from_numpy(scales).cuda(), 4)
    monkeypatch.setenv("CQ_UMMA_GEOMETRY", "prefill")
    pre = lut_gemm_tc(qa, pw, planes, "umma128u").clone()
    monkeypatch.setenv("CQ_UMMA_GEOMETRY", "decode")
    dec = lut_gemm_tc(qa, pw, planes, "umma128u").clone()
    torch.cuda.synchronize()
    assert torch.equal(pre, dec)
    want = oracle.c_lut_gemm(codes, scales, ids, cent, g)
    assert o.relative_error(pre.cpu().numpy(), want) <= (2e-6 if planes == 3 else 2e-4)


def test_prefill_moe_layer_bitwise_equals_decode(monkeypatch):
    """A prefill-sized MoE layer (avg 200 routes per expert): the grouped
    prefill GEMMs (stream-K tail included) equal the decode geometry bitwise."""
    n, d, ff, E, k, g = 400, 1024, 1536, 4, 2, 128
    v, w, sites, _ = moe_inputs_device(43, n, d, ff, E, g)
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, path="tc")
    layer.prepare_tc()
    monkeypatch.setenv("CQ_UMMA_GEOMETRY", "prefill")
    pre = layer(v).clone()
    monkeypatch.setenv("CQ_UMMA_GEOMETRY", "decode")
    dec = layer(v).clone()
    torch.cuda.synchronize()
    assert torch.equal(pre, dec)


@pytest.mark.parametrize("layout", ["umma128u"])
@pytest.mark.parametrize("n,d_in,d_out,g", [(5, 1024, 512, 128), (300, 2048, 768, 128)])
def test_a8_codes_tensor_core_vs_reference_gemm(layout, n, d_in, d_out, g):
    """A8 (8-bit activation codes): the tensor-core kernel with
    codes in [-128, 127] matches the ordered reference_gemm chain within the
    3-plane digit tolerance."""
    rng = np.random.default_rng(n * 7 + d_in)
    cent, ids, pw = _rand_pw(rng, d_out, d_in, g)
    codes = rng.integers(-128, 128, (n, d_in)).astype(np.int8)
    scales = (0.01 + 0.02 * rng.random(n)).astype(np.float32)
    want = oracle.c_lut_gemm(codes, scales, ids, cent, g, table=False)
    qa = QuantizedActivations(torch.from_numpy(codes).cuda(), torch.from_numpy(scales).cuda(), 8)
    got = lut_gemm_tc(qa, pw, 3, layout).cpu().numpy()
    assert o.relative_error(got, want) <= 2e-6


def _pw_k(rng, d_out, d_in, g, kc):
    """A K = kc codebook in the reference's packed format (centroids zero-padded to 16)."""
    cent = (rng.standard_normal((d_out, d_in // g, 16)) * 0.05).astype(np.float32)
    cent[:, :, kc:] = 0.0
    ids = rng.integers(0, kc, (d_out, d_in)).astype(np.uint8)
    packed = (ids[:, 0::2] | (ids[:, 1::2] << 4)).astype(np.uint8)
    return cent, packed, PackedClusteredWeights(torch.from_numpy(cent), torch.from_numpy(packed), d_in, g)


@pytest.mark.parametrize("kc", [4, 8])
@pytest.mark.parametrize("n,d_in,d_out,planes", [(9, 1024, 512, 3), (300, 2048, 768, 3), (40, 1024, 256, 2)])
def test_narrow_codebooks_single_prmt_bitwise_equals_wide(monkeypatch, kc, n, d_in, d_out, planes):
    """K <= 8 codebooks (W3 / W2): prepare_tc selects the
    single-PRMT lookup (umma128u8) from the data; on the same prepared tables it
    is bitwise equal to the 16-entry lookup, and within the plane tolerance of
    the ordered reference GEMM."""
    rng = np.random.default_rng(kc * 100 + n)
    cent, packed, pw = _pw_k(rng, d_out, d_in, 128, kc)
    codes = rng.integers(-8, 8, (n, d_in)).astype(np.int8)
    scales = (rng.random(n) + 0.5).astype(np.float32)
    qa = QuantizedActivations(torch.from_numpy(codes).cuda(), torch.from_numpy(scales).cuda(), 4)
    pw.prepare_tc(planes, "umma128u")
    assert pw.tc["kernel_layout"] == "umma128u8"
    narrow = lut_gemm_tc(qa, pw, planes, "umma128u")
    monkeypatch.setenv("CQ_NARROW", "0")
    _, _, wide_pw = _pw_k(np.random.default_rng(kc * 100 + n), d_out, d_in, 128, kc)
    wide_pw.prepare_tc(planes, "umma128u")
    assert wide_pw.tc["kernel_layout"] == "umma128u"
    wide = lut_gemm_tc(qa, wide_pw, planes, "umma128u")
    assert torch.equal(narrow, wide)
    want = oracle.c_lut_gemm(codes, scales, packed, cent, 128)
    assert o.relative_error(narrow.cpu().numpy(), want) <= (2e-6 if planes == 3 else 2e-4)


def test_narrow_ids_detection_rejects_wide_codebooks():
    rng = np.random.default_rng(3)
    _, _, pw = _pw_k(rng, 128, 256, 128, 8)
    ids = pw.ids_packed.clone()
    ids[5, 7] |= 0x80  # one id 8 or more
    pw2 = PackedClusteredWeights(pw.centroids, ids, 256, 128)
    pw2.prepare_tc(3, "umma128u")
    assert pw2.tc["kernel_layout"] == "umma128u"


@pytest.mark.parametrize("kc", [4, 8])
def test_w3_w2_moe_layer_tc_vs_oracle_and_wide(monkeypatch, kc):
    """A MoE layer whose codebooks all have K = kc: the narrow kernels for
    gate|up and down, against the composed CPU oracle and bitwise against the
    16-entry lookup."""
    n, d, ff, E, k, g = 40, 512, 384, 8, 2, 128
    v, w, sites, _ = moe_inputs_device(kc + 5, n, d, ff, E, g, kc=kc)
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, path="tc")
    layer.prepare_tc()
    assert all(s.tc["kernel_layout"] == "umma128u8" for s in stacks)
    out = layer(v).clone()
    monkeypatch.setenv("CQ_NARROW", "0")
    stacks_w = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    wide = MoELayer.from_stacks(w, *stacks_w, top_k=k, path="tc")
    wide.prepare_tc()
    assert all(s.tc["kernel_layout"] == "umma128u" for s in stacks_w)
    assert torch.equal(wide(v), out)
    host = [[(sites[s][1][e].cpu().numpy(), sites[s][0][e].cpu().numpy(), g) for s in ("gate", "up", "down")]
            for e in range(E)]
    want = oracle.moe_layer_fast(v.float().cpu().numpy(), w.cpu().numpy(), host, k)
    assert o.relative_error(out.cpu().numpy(), want) <= 1e-2
