"""GPU parity of the single operators against the oracle / golden vectors.

Bit-exact: quantizer, nibble unpack, ordered reference GEMM (== the
reference's lut_gemm bits), ordered matmul, top-k ids.  Tolerance: the fp32
LUT GEMM (FMA, warp-split accumulation) <= 1e-6 relative (Frobenius) and the
tensor-core path <= 1e-5 (int8 digit planes)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import oracle as o  # noqa: E402
from paper_2604_10496_b200 import (QuantizedActivations, QuantSpec, kernels, lut_gemm,  # noqa: E402
                                   pack_weights, quantize_activations, reference_gemm)
from paper_2604_10496_b200.errors import ConfigError, DivergenceError, ShapeError  # noqa: E402
from paper_2604_10496_b200.lutgemm import PackedClusteredWeights  # noqa: E402


def _pw(ids, cent, d_in, g):
    return PackedClusteredWeights(torch.from_numpy(cent), torch.from_numpy(ids), d_in, g)


def _qa(codes, scales, bits=4):
    return QuantizedActivations(torch.from_numpy(codes).cuda(), torch.from_numpy(scales).cuda(), bits)


def test_quantizer_bit_exact_golden(golden):
    g = golden("quant.npz")
    n = 0
    for key in sorted({k.rsplit("_", 1)[0] for k in g if k.endswith("_x")}):
        x = g[key + "_x"]
        if x.dtype != np.float32:
            continue
        qa = quantize_activations(torch.from_numpy(x))
        assert np.array_equal(qa.codes.cpu().numpy(), g[key + "_codes"]), key
        assert np.array_equal(qa.scales.cpu().numpy().view(np.uint32), g[key + "_scales"].view(np.uint32)), key
        n += 1
    assert n >= 7


def test_quantizer_bf16_and_random_rows():
    rng = np.random.default_rng(3)
    for n, d, mag in ((1, 7, 1.0), (257, 1024, 3.0), (64, 14336, 0.05), (5, 4096, 1e4)):
        x = (rng.standard_normal((n, d)) * mag).astype(np.float32)
        x[0, : min(d, 8)] = np.array([0.5, -0.5, 1.5, 2.5, -3.5, 7.0, 0, 6.5])[: min(d, 8)]
        xb = torch.from_numpy(x).to(torch.bfloat16)
        want_c, want_s = oracle.c_quantize(xb.float().numpy())
        qa = quantize_activations(xb.cuda())
        assert np.array_equal(qa.codes.cpu().numpy(), want_c)
        assert np.array_equal(qa.scales.cpu().numpy().view(np.uint32), want_s.view(np.uint32))


def test_quantizer_errors():
    with pytest.raises(DivergenceError):
        quantize_activations(torch.tensor([[1.0, float("inf")]]))
    with pytest.raises(ShapeError):
        quantize_activations(torch.zeros(3))
    with pytest.raises(ConfigError):
        quantize_activations(torch.zeros((2, 2)), QuantSpec(8))


def test_unpack_ids_bit_exact():
    rng = np.random.default_rng(4)
    for rows, d_in in ((3, 1), (6, 15), (64, 4096), (7, 45)):
        packed = rng.integers(0, 256, (rows, (d_in + 1) // 2)).astype(np.uint8)
        got = kernels.unpack_ids(torch.from_numpy(packed).cuda(), d_in).cpu().numpy()
        assert np.array_equal(got, o.unpack_ids(packed, d_in))
    every = np.arange(256, dtype=np.uint8)[None, :]
    got = kernels.unpack_ids(torch.from_numpy(every).cuda(), 512).cpu().numpy()
    assert np.array_equal(o.pack_ids(got), every)


def _cases(g):
    for i in range(int(g["count"])):
        k = f"c{i:03d}"
        d_in, gs = (int(v) for v in g[k + "_meta"])
        yield str(g[k + "_tag"]), g[k + "_codes"], g[k + "_scales"], g[k + "_ids"], g[k + "_cent"], d_in, gs, g[k + "_out"]


def test_reference_gemm_bit_exact_golden(golden):
    g = golden("lutgemm.npz")
    for tag, codes, scales, ids, cent, d_in, gs, want in _cases(g):
        got = reference_gemm(_qa(codes, scales), _pw(ids, cent, d_in, gs)).cpu().numpy()
        assert np.array_equal(got.view(np.int32), want.view(np.int32)), tag


def test_eight_bit_codes_bit_exact(golden):
    g = golden("lutgemm.npz")
    got = reference_gemm(_qa(g["a8_codes"], g["a8_scales"], 8), _pw(g["a8_ids"], g["a8_cent"], 32, 16))
    assert np.array_equal(got.cpu().numpy().view(np.int32), g["a8_out"].view(np.int32))


def test_lut_gemm_golden_within_tolerance(golden):
    g = golden("lutgemm.npz")
    for tag, codes, scales, ids, cent, d_in, gs, want in _cases(g):
        got = lut_gemm(_qa(codes, scales), _pw(ids, cent, d_in, gs)).cpu().numpy()
        assert o.relative_error(got, want) <= 1e-6, tag
        if not want.any():
            assert not got.any(), tag


def test_lut_gemm_matches_oracle_full_size():
    rng = np.random.default_rng(7)
    for n, d_in, d_out, g in ((1, 4096, 1024, 128), (16, 4096, 2048, 128), (64, 1024, 2816, 128),
                              (33, 2048, 768, 2048), (5, 512, 96, 32)):
        codes = rng.integers(-8, 8, (n, d_in)).astype(np.int8)
        scales = (0.5 + rng.random(n)).astype(np.float32)
        cent = rng.standard_normal((d_out, d_in // g, 16)).astype(np.float32)
        ids = rng.integers(0, 256, (d_out, d_in // 2)).astype(np.uint8)
        want = oracle.c_lut_gemm(codes, scales, ids, cent, g)
        pw = _pw(ids, cent, d_in, g)
        got = lut_gemm(_qa(codes, scales), pw).cpu().numpy()
        # fp32 accumulation-order noise grows ~sqrt(d_in): 3e-6 at d_in = 4096
        assert o.relative_error(got, want) <= 3e-6, (n, d_in, d_out, g)
        exact = reference_gemm(_qa(codes, scales), pw).cpu().numpy()
        assert np.array_equal(exact.view(np.int32), want.view(np.int32)), (n, d_in, d_out, g)


def test_hand_summed_single_token():
    cents = np.zeros((1, 1, 16))
    cents[0, 0, :4] = [0.5, -1.0, 2.0, 0.25]
    pw = pack_weights(cents, np.array([[0, 1, 2, 3]], dtype=np.uint8), None)
    qa = _qa(np.array([[3, -8, 1, 4]], np.int8), np.array([1.0], np.float32))
    want = np.float32(0.5 * 3 + (-1.0) * (-8) + 2.0 * 1 + 0.25 * 4)
    assert lut_gemm(qa, pw).item() == want
    assert reference_gemm(qa, pw).item() == want


def test_zero_activations_zero_output():
    rng = np.random.default_rng(8)
    pw = pack_weights(rng.standard_normal((16, 2, 16)), rng.integers(0, 16, (16, 64)).astype(np.uint8), 32)
    qa = _qa(np.zeros((5, 64), np.int8), np.ones(5, np.float32))
    assert not lut_gemm(qa, pw).any() and not reference_gemm(qa, pw).any()


def test_empty_and_validation():
    rng = np.random.default_rng(9)
    pw = pack_weights(rng.standard_normal((8, 1, 16)), rng.integers(0, 16, (8, 16)).astype(np.uint8), None)
    out = lut_gemm(_qa(np.zeros((0, 16), np.int8), np.zeros(0, np.float32)), pw)
    assert out.shape == (0, 8)
    with pytest.raises(ConfigError, match="4-bit"):
        lut_gemm(_qa(np.zeros((1, 16), np.int8), np.ones(1, np.float32), 8), pw)
    with pytest.raises(ConfigError, match="token block"):
        lut_gemm(_qa(np.zeros((1, 16), np.int8), np.ones(1, np.float32)), pw, block_tokens=0)
    with pytest.raises(ShapeError, match="dim"):
        lut_gemm(_qa(np.zeros((1, 32), np.int8), np.ones(1, np.float32)), pw)
    with pytest.raises(ShapeError, match="scales"):
        reference_gemm(QuantizedActivations(torch.zeros((2, 16), dtype=torch.int8).cuda(),
                                            torch.ones(1).cuda(), 4), pw)


def test_block_and_thread_arguments_do_not_change_results():
    rng = np.random.default_rng(10)
    pw = pack_weights(rng.standard_normal((48, 6, 16)), rng.integers(0, 16, (48, 48)).astype(np.uint8), 8)
    qa = quantize_activations(torch.from_numpy(rng.standard_normal((70, 48)).astype(np.float32)))
    base = lut_gemm(qa, pw)
    for bt, th in ((1, 1), (17, 3), (4096, 8)):
        assert torch.equal(lut_gemm(qa, pw, block_tokens=bt, threads=th), base)


def test_matmul_and_topk_bit_exact(golden):
    g = golden("routing.npz")
    a, b = torch.from_numpy(g["mm_a"]).cuda(), torch.from_numpy(g["mm_b"]).cuda()
    out = torch.empty((a.shape[0], b.shape[1]), device="cuda")
    kernels.matmul_into(a, b, out)
    assert np.array_equal(out.cpu().numpy().view(np.int32), g["mm_out"].view(np.int32))
    from paper_2604_10496_b200 import _lib
    for k in (1, 2, 6):
        logits = torch.from_numpy(g["mm_out"]).cuda()
        sel = torch.empty((logits.shape[0], k), dtype=torch.int32, device="cuda")
        w = torch.empty((logits.shape[0], k), dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().cq_route_topk(logits.data_ptr(), logits.shape[0], logits.shape[1], k,
                                            sel.data_ptr(), w.data_ptr(), _lib.stream()))
        assert np.array_equal(sel.cpu().numpy(), g[f"topk{k}_sel"])
        ulp = np.abs(w.cpu().numpy().view(np.int32) - g[f"topk{k}_w"].view(np.int32))
        assert ulp.max() <= 8  # CUDA expf vs numpy float32 exp: ulp-bounded
    ties = torch.from_numpy(g["ties_logits"]).cuda()
    sel = torch.empty((3, 2), dtype=torch.int32, device="cuda")
    w = torch.empty((3, 2), device="cuda")
    _lib.check(_lib.lib().cq_route_topk(ties.data_ptr(), 3, 4, 2, sel.data_ptr(), w.data_ptr(), _lib.stream()))
    assert np.array_equal(sel.cpu().numpy(), g["ties_sel"])
