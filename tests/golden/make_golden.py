"""Generate the golden fixtures that pin the oracle — run HERE, where the
read-only reference is mounted (it is not present on the GPU box).

    python tests/golden/make_golden.py

Imports the reference package from /root/reference/pkg/src with its numpy
backend (CODEQUANT_BACKEND=python; bitwise identical to the compiled one,
reference tests/test_lutgemm.py:215-230) and records inputs + outputs of the
reference's own functions on the path:

  quant.npz    quantize_activations (quant.py:89-100): hand rows of
               tests/test_quant.py:19-36, exact .5 ties, zero rows, fp32/fp64.
  lutgemm.npz  lut_gemm / reference_gemm (lutgemm.py:133-161) on the sweep of
               tests/test_lutgemm.py:167-184 (odd d_in, g=9, g=d_in, zero rows),
               acceptance #8 style K=5 cases (tests/test_acceptance.py:358-387),
               the hand-summed token (tests/test_lutgemm.py:112-120) and 8-bit codes.
  routing.npz  linalg.matmul fp32 (linalg.py:66-75) and select_top_k
               (model.py:324-330) incl. exact ties (tests/test_model.py:301-305).
  acceptance8.npz  the 216 instances of acceptance criterion #8
               (tests/test_acceptance.py:358-387): the instance parameters and a
               SHA-256 of the reference's reference_gemm output bytes (and of its
               codes / scales), so the GPU test can regenerate the inputs with the
               same numpy draws and check the backend bytewise without shipping
               the arrays.
  moe_*.npz    the MoE block composed from reference functions:
               quantize_activations -> matmul(router) -> select_top_k ->
               per expert ascending lut_gemm(gate/up) -> silu*up ->
               quantize_activations -> lut_gemm(down) -> weighted sum.
               Inputs are regenerated from seeds by the package's synthetic
               generator; the fixture stores a SHA-256 of those inputs as made
               here with the reference's RngState, so the test proves both the
               generator and the outputs.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

os.environ["CODEQUANT_BACKEND"] = "python"
sys.path.insert(0, "/root/reference/pkg/src")

from codequant.linalg import RngState, matmul  # noqa: E402
from codequant.lutgemm import lut_gemm, pack_weights, reference_gemm  # noqa: E402
from codequant.model import select_top_k, silu  # noqa: E402
from codequant.quant import QuantizedActivations, QuantSpec, quantize_activations  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays)
    print("wrote", name, sum(a.nbytes for a in arrays.values() if hasattr(a, "nbytes")), "bytes raw")


def make_quant():
    rows = []
    rows.append(np.array([[1.0, 2.0, 3.5]]))                     # test_quant.py:19-22
    rows.append(np.array([[7.0, -7.0, 0.0]]))                    # :25-30
    rows.append(np.zeros((1, 3)))                                # :33-36
    rows.append(np.array([[0.5, 1.5, 2.5, -0.5, -2.5, 3.5, -3.5, 7.0]]))  # .5 ties at s=1
    rng = np.random.default_rng(11)
    cases = {}
    for i, r in enumerate(rows):
        for dt in (np.float64, np.float32):
            x = r.astype(dt)
            qa = quantize_activations(x, QuantSpec(4))
            cases[f"hand{i}_{np.dtype(dt).name}_x"] = x
            cases[f"hand{i}_{np.dtype(dt).name}_codes"] = qa.codes
            cases[f"hand{i}_{np.dtype(dt).name}_scales"] = qa.scales
    for i, (n, d, mag) in enumerate([(40, 17, 1.0), (64, 256, 3.0), (33, 100, 1e-3),
                                     (16, 1024, 50.0), (8, 31, 1e-30)]):
        for dt in (np.float32, np.float64):
            x = (rng.standard_normal((n, d)) * mag).astype(dt)
            x[0] = 0.0
            if d > 8:
                x[1, :8] = np.array([0.5, 1.5, -2.5, 3.5, 7, -7, 0.25, 6.5]) * (x[1, 8] if n > 1 else 1)
            qa = quantize_activations(x, QuantSpec(4))
            key = f"rand{i}_{np.dtype(dt).name}"
            cases[key + "_x"] = x
            cases[key + "_codes"] = qa.codes
            cases[key + "_scales"] = qa.scales
    save("quant.npz", **cases)


def random_instance(seed, n_tokens, d_in, group_size, k=16, d_out=None, zero_rows=0):
    """tests/test_lutgemm.py:13-24."""
    rng = RngState(seed)
    x = rng.stream("x").standard_normal((n_tokens, d_in)) * 3.0
    if zero_rows:
        x[:zero_rows] = 0.0
    qa = quantize_activations(x, QuantSpec(4))
    d_out = d_in if d_out is None else d_out
    g = d_in if group_size is None else group_size
    cents = rng.stream("c").standard_normal((d_out, d_in // g, k))
    ids = rng.stream("i").integers(0, k, (d_out, d_in)).astype(np.uint8)
    return qa, pack_weights(cents, ids, group_size)


def make_lutgemm():
    cases = {}
    idx = 0

    def add(qa, pw, tag):
        nonlocal idx
        out_l = lut_gemm(qa, pw)
        out_r = reference_gemm(qa, pw)
        assert out_l.tobytes() == out_r.tobytes()
        key = f"c{idx:03d}"
        cases[key + "_codes"] = qa.codes.astype(np.int8)
        cases[key + "_scales"] = np.asarray(qa.scales, np.float32)
        cases[key + "_ids"] = pw.ids_packed
        cases[key + "_cent"] = pw.centroids
        cases[key + "_meta"] = np.array([pw.d_in, pw.group_size], np.int64)
        cases[key + "_out"] = out_l
        cases[key + "_tag"] = np.array(tag)
        idx += 1

    case = 0
    for n_tokens in (1, 7, 64):                       # test_lutgemm.py:167-184
        for d_in, gs in ((16, None), (16, 16), (64, 16), (64, 64), (15, None), (45, 9)):
            case += 1
            qa, pw = random_instance(100 + case, n_tokens, d_in, gs, zero_rows=case % 3 == 0)
            add(qa, pw, f"sweep n={n_tokens} d={d_in} g={gs}")
    for seed in range(2):                              # acceptance #8 style, K=5 / 16
        for n, d in ((7, 64), (64, 256), (256, 64)):
            for g in sorted({16, 64, d}):
                if g > d:
                    continue
                rng = np.random.default_rng(1_000_003 * seed + 1009 * n + 13 * d + g)
                k = 5 if (n + g) % 3 == 0 else 16
                x = rng.standard_normal((n, d))
                x[: max(1, n // 4)] = 0.0
                qa = quantize_activations(x, QuantSpec(4))
                d_out = 16 if (n + d) % 2 else 8
                cents = rng.standard_normal((d_out, d // g, k)).astype(np.float32)
                ids = rng.integers(0, k, (d_out, d), dtype=np.uint8)
                add(qa, pack_weights(cents, ids, None if g == d else g), f"acc8 n={n} d={d} g={g} k={k}")
    # hand-summed single token (test_lutgemm.py:112-120): 1.5 + 8 + 2 + 1
    cents = np.zeros((1, 1, 16))
    cents[0, 0, :4] = [0.5, -1.0, 2.0, 0.25]
    pw = pack_weights(cents, np.array([[0, 1, 2, 3]], dtype=np.uint8), None)
    qa = QuantizedActivations(np.array([[3, -8, 1, 4]], np.int8), np.array([1.0], np.float32), 4)
    add(qa, pw, "hand single token")
    # full code range incl. -8 (bench draws U[-8,8), lutgemm.py:216)
    rng = np.random.default_rng(5)
    codes = rng.integers(-8, 8, (9, 256)).astype(np.int8)
    scales = (0.5 + rng.random(9)).astype(np.float32)
    cents = rng.standard_normal((24, 2, 16))
    ids = rng.integers(0, 16, (24, 256)).astype(np.uint8)
    add(QuantizedActivations(codes, scales, 4), pack_weights(cents, ids, 128), "bench-range codes")
    # 8-bit codes through reference_gemm (test_lutgemm.py:152-164)
    rng8 = RngState(13)
    x8 = rng8.stream("x").standard_normal((6, 32))
    qa8 = quantize_activations(x8, QuantSpec(8))
    pw8 = pack_weights(rng8.stream("c").standard_normal((8, 2, 16)),
                       rng8.stream("i").integers(0, 16, (8, 32)).astype(np.uint8), 16)
    cases["a8_codes"] = qa8.codes
    cases["a8_scales"] = qa8.scales.astype(np.float32)
    cases["a8_ids"] = pw8.ids_packed
    cases["a8_cent"] = pw8.centroids
    cases["a8_out"] = reference_gemm(qa8, pw8)
    cases["count"] = np.array(idx)
    save("lutgemm.npz", **cases)


def make_routing():
    rng = RngState(21)
    a = rng.stream("a").standard_normal((37, 300)).astype(np.float32)
    b = rng.stream("b").standard_normal((300, 16)).astype(np.float32)
    logits = matmul(a, b)
    cases = dict(mm_a=a, mm_b=b, mm_out=logits)
    for k in (1, 2, 6):
        sel, w = select_top_k(logits, k)
        cases[f"topk{k}_sel"] = sel
        cases[f"topk{k}_w"] = w
    ties = np.zeros((3, 4), np.float32)
    ties[1] = [1.0, 2.0, 2.0, 1.0]
    ties[2] = [-0.0, 0.0, -1.0, 0.0]
    sel, w = select_top_k(ties, 2)
    cases.update(ties_logits=ties, ties_sel=sel, ties_w=w)
    save("routing.npz", **cases)


def synth_inputs(seed, n, d, ff, n_exp, g):
    """The synthetic MoE inputs of SURVEY §8(d), drawn with the REFERENCE's
    RngState.  Mirrored by paper_2604_10496_b200.synthetic.moe_inputs."""
    rng = RngState(seed)
    v = rng.stream("moe.v").standard_normal((n, d)).astype(np.float32)
    # round to bf16 (round-to-nearest-even), then the exact fp32 upcast
    bits = v.view(np.uint32).astype(np.uint64)
    bits = ((bits + 0x7FFF + ((bits >> 16) & 1)) >> 16) << 16
    v = bits.astype(np.uint32).view(np.float32)
    w_router = (rng.stream("moe.router").standard_normal((d, n_exp)) / np.sqrt(d)).astype(np.float32)
    experts = []
    for e in range(n_exp):
        mats = []
        for site, (di, do) in (("gate", (d, ff)), ("up", (d, ff)), ("down", (ff, d))):
            cents = (rng.stream(f"moe.e{e}.{site}.c").standard_normal((do, di // g, 16))
                     / np.sqrt(di)).astype(np.float32)
            ids = rng.stream(f"moe.e{e}.{site}.i").integers(0, 16, (do, di)).astype(np.uint8)
            mats.append(pack_weights(cents, ids, g))
        experts.append(mats)
    return v, w_router, experts


def input_digest(v, w_router, experts) -> str:
    h = hashlib.sha256()
    h.update(v.tobytes())
    h.update(w_router.tobytes())
    for mats in experts:
        for pw in mats:
            h.update(pw.centroids.tobytes())
            h.update(pw.ids_packed.tobytes())
    return h.hexdigest()


def reference_moe(v, w_router, experts, top_k):
    """SURVEY §8(c) recipe on reference functions only."""
    n = v.shape[0]
    qa = quantize_activations(v, QuantSpec(4))
    router_in = qa.codes.astype(np.float32) * qa.scales[:, None]
    logits = matmul(router_in, w_router)
    sel, wts = select_top_k(logits, top_k)
    dense = np.zeros((n, len(experts)), np.float32)
    np.put_along_axis(dense, sel, wts, axis=1)
    out = np.zeros_like(v)
    for e, (gate, up, down) in enumerate(experts):
        rows = np.nonzero((sel == e).any(axis=1))[0]
        if rows.size == 0:
            continue
        sub = QuantizedActivations(qa.codes[rows], qa.scales[rows], 4)
        a = lut_gemm(sub, gate)
        b = lut_gemm(sub, up)
        h = silu(a) * b
        f = lut_gemm(quantize_activations(h, QuantSpec(4)), down)
        out[rows] = out[rows] + dense[rows, e, None] * f
    return out, logits, sel, wts, qa


def make_moe(name, seed, n, d, ff, n_exp, top_k, g):
    v, w_router, experts = synth_inputs(seed, n, d, ff, n_exp, g)
    out, logits, sel, wts, qa = reference_moe(v, w_router, experts, top_k)
    save(name, digest=np.array(input_digest(v, w_router, experts)),
         config=np.array([seed, n, d, ff, n_exp, top_k, g], np.int64),
         out=out, logits=logits, selected=sel, weights=wts,
         codes=qa.codes, scales=qa.scales)


def acceptance8_instances():
    """Yields the exact inputs of tests/test_acceptance.py:358-387 (same rng
    draws, same order) plus the instance parameters."""
    from itertools import product
    combos = [(n, d, g) for n, d in product((1, 7, 64, 256), (16, 64, 256)) for g in sorted({16, 64, d}) if g <= d]
    instances = 0
    for seed in range(9):
        for n_tokens, d_in, g in combos:
            rng = np.random.default_rng(1_000_003 * seed + 1009 * n_tokens + 13 * d_in + g)
            d_out = 16 if instances % 2 else 8
            k = 16 if instances % 3 else 5
            x = rng.standard_normal((n_tokens, d_in))
            if instances % 3 == 0:
                x[: max(1, n_tokens // 4)] = 0.0  # all-zero rows
            centroids = rng.standard_normal((d_out, d_in // g, k)).astype(np.float32)
            ids = rng.integers(0, k, (d_out, d_in), dtype=np.uint8)
            yield (seed, n_tokens, d_in, g, d_out, k), x, centroids, ids
            instances += 1


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_acceptance8():
    params, out_sha, codes_sha, scales_sha = [], [], [], []
    for p, x, centroids, ids in acceptance8_instances():
        seed, n_tokens, d_in, g, d_out, k = p
        qa = quantize_activations(x, QuantSpec(4))
        pw = pack_weights(centroids, ids, None if g == d_in else g)
        want = reference_gemm(qa, pw)
        assert lut_gemm(qa, pw).tobytes() == want.tobytes()
        params.append(p)
        out_sha.append(sha(want))
        codes_sha.append(sha(qa.codes))
        scales_sha.append(sha(qa.scales.astype(np.float32)))
    save("acceptance8.npz", params=np.array(params, np.int64), out_sha=np.array(out_sha),
         codes_sha=np.array(codes_sha), scales_sha=np.array(scales_sha))


def make_rng():
    r = RngState(1234)
    save("rng.npz", normal=r.stream("t", 3).standard_normal(8),
         ints=r.stream("u").integers(0, 16, 16))


if __name__ == "__main__":
    if sys.argv[1:] == ["acceptance8"]:  # just the new fixture (the others are byte-stable in git)
        make_acceptance8()
        sys.exit(0)
    make_acceptance8()
    make_rng()
    make_quant()
    make_lutgemm()
    make_routing()
    make_moe("moe_small.npz", 3, 24, 64, 96, 4, 2, 32)
    make_moe("moe_odd.npz", 4, 9, 128, 160, 6, 3, 32)
    make_moe("moe_c1.npz", 0, 64, 1024, 2816, 8, 2, 128)   # config 1, full size
