"""Pin the CPU oracle (numpy + C restatements) to the reference's own outputs.

Golden fixtures come from tests/golden/make_golden.py, which imports the
read-only reference.  These tests run on CPU only."""

import os

import numpy as np
import pytest

import oracle
from oracle import oracle as o


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build(ref=os.path.exists("/root/reference"))


def test_rng_matches_reference(golden):
    g = golden("rng.npz")
    r = o.RngState(1234)
    assert np.array_equal(r.stream("t", 3).standard_normal(8), g["normal"])
    assert np.array_equal(r.stream("u").integers(0, 16, 16), g["ints"])


def _quant_cases(g):
    keys = sorted({k.rsplit("_", 1)[0] for k in g if k.endswith("_x")})
    for key in keys:
        yield key, g[key + "_x"], g[key + "_codes"], g[key + "_scales"]


def test_quantize_matches_golden(golden):
    g = golden("quant.npz")
    n = 0
    for key, x, codes, scales in _quant_cases(g):
        q, s = o.quantize(x, 4)
        assert np.array_equal(q, codes), key
        assert s.dtype == scales.dtype and np.array_equal(s.view(np.uint8), scales.view(np.uint8)), key
        n += 1
    assert n >= 16


def test_c_quantize_matches_golden_f32(golden):
    g = golden("quant.npz")
    for key, x, codes, scales in _quant_cases(g):
        if x.dtype != np.float32:
            continue
        q, s = oracle.c_quantize(x)
        assert np.array_equal(q, codes), key
        assert np.array_equal(s.view(np.uint32), scales.view(np.uint32)), key


def test_quantize_hand_rows(golden):
    q, s = o.quantize(np.array([[1.0, 2.0, 3.5]]))
    assert s[0] == 0.5 and q.tolist() == [[2, 4, 7]]
    q, s = o.quantize(np.zeros((1, 5)))
    assert s[0] == 1.0 and not q.any()


def _gemm_cases(g):
    for i in range(int(g["count"])):
        key = f"c{i:03d}"
        d_in, gs = (int(v) for v in g[key + "_meta"])
        yield (key, str(g[key + "_tag"]), g[key + "_codes"], g[key + "_scales"], g[key + "_ids"],
               g[key + "_cent"], d_in, gs, g[key + "_out"])


def test_lut_gemm_bitwise_golden(golden):
    g = golden("lutgemm.npz")
    for key, tag, codes, scales, ids, cent, d_in, gs, want in _gemm_cases(g):
        got = o.lut_gemm(codes, scales, ids, cent, gs)
        assert np.array_equal(got.view(np.int32), want.view(np.int32)), tag
        got_r = o.reference_gemm(codes, scales, ids, cent, gs)
        assert np.array_equal(got_r.view(np.int32), want.view(np.int32)), tag


def test_c_lut_gemm_bitwise_golden(golden):
    g = golden("lutgemm.npz")
    for key, tag, codes, scales, ids, cent, d_in, gs, want in _gemm_cases(g):
        for table in (True, False):
            got = oracle.c_lut_gemm(codes, scales, ids, cent, gs, threads=3, table=table)
            assert np.array_equal(got.view(np.int32), want.view(np.int32)), (tag, table)


def test_hand_summed_token(golden):
    # reference tests/test_lutgemm.py:112-120: 0.5*3 + (-1)*(-8) + 2*1 + 0.25*4
    g = golden("lutgemm.npz")
    tags = {str(g[f"c{i:03d}_tag"]): f"c{i:03d}" for i in range(int(g["count"]))}
    key = tags["hand single token"]
    assert g[key + "_out"][0, 0] == np.float32(0.5 * 3 + (-1.0) * (-8) + 2.0 * 1 + 0.25 * 4)


def test_eight_bit_reference_golden(golden):
    g = golden("lutgemm.npz")
    got = o.reference_gemm(g["a8_codes"], g["a8_scales"], g["a8_ids"], g["a8_cent"], 16)
    assert np.array_equal(got.view(np.int32), g["a8_out"].view(np.int32))


def test_matmul_and_topk_golden(golden):
    g = golden("routing.npz")
    got = o.matmul_ordered(g["mm_a"], g["mm_b"])
    assert np.array_equal(got.view(np.int32), g["mm_out"].view(np.int32))
    assert np.array_equal(oracle.c_matmul(g["mm_a"], g["mm_b"]).view(np.int32), g["mm_out"].view(np.int32))
    for k in (1, 2, 6):
        sel, w = o.select_top_k(g["mm_out"], k)
        assert np.array_equal(sel, g[f"topk{k}_sel"])
        assert np.array_equal(w, g[f"topk{k}_w"])
    sel, w = o.select_top_k(g["ties_logits"], 2)
    assert np.array_equal(sel, g["ties_sel"]) and np.array_equal(w, g["ties_w"])


def test_route_permutation_properties():
    rng = np.random.default_rng(0)
    sel = np.stack([rng.permutation(8)[:3] for _ in range(50)])
    tok, slot, off, inv = o.route_permutation(sel, 8)
    assert off[-1] == sel.size and np.all(np.diff(off) >= 0)
    for e in range(8):
        seg = tok[off[e]:off[e + 1]]
        assert np.all(np.diff(seg) > 0)                      # tokens ascending in a segment
        assert np.all(sel[seg, slot[off[e]:off[e + 1]]] == e)
    assert np.array_equal(np.sort(inv.reshape(-1)), np.arange(sel.size))


def _moe_from_golden(g):
    from paper_2604_10496_b200.synthetic import input_digest, moe_inputs_host
    seed, n, d, ff, E, k, gs = (int(v) for v in g["config"])
    v, w, experts, _ = moe_inputs_host(seed, n, d, ff, E, gs)
    assert input_digest(v, w, experts) == str(g["digest"]), "synthetic generator drifted from golden"
    return v, w, experts, k


@pytest.mark.parametrize("name", ["moe_small.npz", "moe_odd.npz"])
def test_moe_oracle_matches_reference_composition(golden, name):
    g = golden(name)
    v, w, experts, k = _moe_from_golden(g)
    out, tr = o.moe_layer(v, w, experts, k, return_trace=True)
    assert np.array_equal(tr["codes"], g["codes"])
    assert np.array_equal(tr["logits"].view(np.int32), g["logits"].view(np.int32))
    assert np.array_equal(tr["selected"], g["selected"])
    assert np.array_equal(tr["weights"], g["weights"])
    assert np.array_equal(out.view(np.int32), g["out"].view(np.int32))


def test_moe_c1_fast_oracle_bitwise(golden):
    g = golden("moe_c1.npz")
    v, w, experts, k = _moe_from_golden(g)
    out = oracle.moe_layer_fast(v, w, experts, k)
    assert np.array_equal(out.view(np.int32), g["out"].view(np.int32))


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(oracle.__file__), "_ref")),
                    reason="reference kernel not built here")
def test_reference_core_agrees_with_restatement(golden):
    g = golden("lutgemm.npz")
    for key, tag, codes, scales, ids, cent, d_in, gs, want in _gemm_cases(g):
        if ids.shape[1] * 2 != d_in and d_in % 2 == 0:
            continue
        got = oracle.ref_lut_gemm(codes, scales, ids, cent, gs, block_tokens=17, threads=2)
        assert np.array_equal(got.view(np.int32), want.view(np.int32)), tag
    gm = golden("moe_small.npz")
    v, w, experts, k = _moe_from_golden(gm)
    out = oracle.moe_layer_reference(v, w, experts, k, threads=2)
    assert np.array_equal(out.view(np.int32), gm["out"].view(np.int32))
