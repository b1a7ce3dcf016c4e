"""CPU oracle for the Stage-4 LUT MoE path — TEST INFRASTRUCTURE ONLY.

This module restates, in numpy, the reference algorithm of CodeQuant's
Stage-4 path (arxiv 2604.10496, reference tree `pkg/src/codequant/`).  It is
the *checker*: only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import it.  The product package
`paper_2604_10496_b200` never imports anything under `oracle/`.

Parity is pinned: `tests/test_oracle.py` checks every function here against
golden vectors produced by the reference itself (`tests/golden/make_golden.py`
imports the read-only reference and commits `tests/golden/*.npz`).

Arithmetic contract restated (reference file:line):
  * quantizer: `quant.py:69-100` — per-row max|x|, scale = max/qmax in the
    input dtype, 3 (= bits-1) low significand bits truncated, scale 1 for an
    all-zero row, round half away from zero, clip to [qmin, qmax].
  * lut / reference GEMM: `kernels/fallback.py:45-80`, `kernels/_core.pyx:41-211`
    — fp32, one rounding per multiply and per add, j ascending, the per-token
    scale multiplied once at the end.  Table entry = centroid * float(code).
  * ordered matmul: `kernels/fallback.py:14-20`, `_core.pyx:27-38` — k ascending.
  * routing: `model.py:324-330` (stable argsort of -logits, softmax over the
    selected logits, `model.py:240-243`).
  * MoE block: `model.py:377-404` composed as SURVEY.md §8(c).
"""

from __future__ import annotations

import hashlib

import numpy as np

TABLE_SIZE = 16


# ---------------------------------------------------------------------------
# Seeded inputs (restates linalg.RngState, linalg.py:32-53)


class RngState:
    """Philox substreams keyed by SHA-256(f"{seed}:{tag}:{index}")[:16]."""

    def __init__(self, seed: int):
        self.seed = int(seed)

    def stream(self, tag: str, index: int = 0) -> np.random.Generator:
        digest = hashlib.sha256(f"{self.seed}:{tag}:{index}".encode()).digest()
        key = np.frombuffer(digest[:16], dtype=np.uint64)
        return np.random.Generator(np.random.Philox(key=key))


# ---------------------------------------------------------------------------
# Quantizer (quant.py:69-100)


def round_half_away(v: np.ndarray) -> np.ndarray:
    t = np.trunc(v)
    return t + np.sign(v) * (np.abs(v - t) >= 0.5)


def snap_scales(scales: np.ndarray, bits: int) -> np.ndarray:
    drop = bits - 1
    s = np.ascontiguousarray(scales)
    if s.dtype == np.float64:
        return (s.view(np.uint64) & ~np.uint64((1 << drop) - 1)).view(np.float64)
    return (s.view(np.uint32) & ~np.uint32((1 << drop) - 1)).view(np.float32)


def quantize(x: np.ndarray, bits: int = 4):
    """Returns (codes int8 (N,d), scales (N,) in x.dtype)."""
    x = np.ascontiguousarray(x)
    qmax = 2 ** (bits - 1) - 1
    qmin = -(2 ** (bits - 1))
    if not np.all(np.isfinite(x)):
        raise FloatingPointError("non-finite activation input to quantizer")
    mx = np.max(np.abs(x), axis=1) if x.shape[1] else np.zeros(x.shape[0], x.dtype)
    s = snap_scales((mx / qmax).astype(x.dtype), bits)
    s = np.where(mx == 0, x.dtype.type(1.0), s)
    q = np.clip(round_half_away(x / s[:, None]), qmin, qmax)
    return q.astype(np.int8), s


# ---------------------------------------------------------------------------
# Packing (lutgemm.py:90-116, fallback.py:35-42)


def pack_ids(ids: np.ndarray) -> np.ndarray:
    """(rows, d_in) ids < 16 -> (rows, ceil(d_in/2)) bytes, low nibble first."""
    ids = np.asarray(ids, dtype=np.uint8)
    if ids.shape[1] % 2:
        ids = np.concatenate([ids, np.zeros((ids.shape[0], 1), np.uint8)], axis=1)
    return (ids[:, 0::2] | (ids[:, 1::2] << np.uint8(4))).astype(np.uint8)


def unpack_ids(ids_packed: np.ndarray, d_in: int) -> np.ndarray:
    out = np.empty((ids_packed.shape[0], ids_packed.shape[1] * 2), np.uint8)
    out[:, 0::2] = ids_packed & np.uint8(0x0F)
    out[:, 1::2] = ids_packed >> np.uint8(4)
    return out[:, :d_in]


def pad_centroids(centroids: np.ndarray) -> np.ndarray:
    d_out, n_groups, k = centroids.shape
    full = np.zeros((d_out, n_groups, TABLE_SIZE), np.float32)
    full[:, :, :k] = centroids
    return full


def build_lut(centroids16: np.ndarray) -> np.ndarray:
    """table[c][a] = c_c * float(a - 8), one fp32 multiply (lutgemm.py:45-50)."""
    c = np.asarray(centroids16, np.float32)
    vals = (np.arange(TABLE_SIZE, dtype=np.int32) - 8).astype(np.float32)
    return c[:, None] * vals[None, :]


# ---------------------------------------------------------------------------
# GEMMs (fallback.py:45-80)


def lut_gemm(codes, scales, ids_packed, centroids, g):
    """y[t,i] = s_t * sum_j table[i, j//g][id][code+8], j ascending, fp32."""
    codes = np.ascontiguousarray(codes, np.int8)
    scales = np.ascontiguousarray(scales, np.float32)
    n, d_in = codes.shape
    d_out = centroids.shape[0]
    acc = np.zeros((n, d_out), np.float32)
    if n == 0 or d_out == 0:
        return acc
    ids = unpack_ids(ids_packed, d_in)
    biased = codes.astype(np.intp) + 8
    vals = (np.arange(TABLE_SIZE, dtype=np.int32) - 8).astype(np.float32)
    tables = centroids[:, :, :, None] * vals          # (d_out, G, 16, 16) fp32
    rows = np.arange(d_out)
    for j in range(d_in):
        tab = tables[rows, j // g, ids[:, j], :]      # (d_out, 16)
        acc += tab[:, biased[:, j]].T
    return scales[:, None] * acc


def reference_gemm(codes, scales, ids_packed, centroids, g):
    """Per-element dequant, same order; bitwise equal to lut_gemm for 4-bit
    codes, and the 8-bit path (lutgemm.py:147-161)."""
    codes = np.ascontiguousarray(codes, np.int8)
    scales = np.ascontiguousarray(scales, np.float32)
    n, d_in = codes.shape
    d_out = centroids.shape[0]
    acc = np.zeros((n, d_out), np.float32)
    if n == 0 or d_out == 0:
        return acc
    ids = unpack_ids(ids_packed, d_in)
    qf = codes.astype(np.float32)
    rows = np.arange(d_out)
    for j in range(d_in):
        cvec = centroids[rows, j // g, ids[:, j]]
        acc += qf[:, j, None] * cvec[None, :]
    return scales[:, None] * acc


def matmul_ordered(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """out[i,j] = (((0 + a[i,0]b[0,j]) + a[i,1]b[1,j]) + ...) in a's dtype."""
    out = np.zeros((a.shape[0], b.shape[1]), a.dtype)
    for k in range(a.shape[1]):
        out += a[:, k, None] * b[k, None, :]
    return out


def dense_weight(centroids, ids_packed, d_in, g) -> np.ndarray:
    """(d_in, d_out) reconstruction (model.py:123-135)."""
    ids = unpack_ids(ids_packed, d_in)
    grp = (np.arange(d_in) // g)[None, :]
    return np.ascontiguousarray(
        centroids[np.arange(centroids.shape[0])[:, None], grp, ids].T)


# ---------------------------------------------------------------------------
# MoE block semantics (model.py:233-243, 324-330, 377-404)


def silu(x: np.ndarray) -> np.ndarray:
    pos = x >= 0
    ex = np.exp(np.where(pos, -x, x))
    return x * np.where(pos, 1.0 / (1.0 + ex), ex / (1.0 + ex))


def softmax(v: np.ndarray, axis: int = -1) -> np.ndarray:
    e = np.exp(v - np.max(v, axis=axis, keepdims=True))
    return e / np.sum(e, axis=axis, keepdims=True)


def select_top_k(logits: np.ndarray, k: int):
    order = np.argsort(-logits, axis=1, kind="stable")
    sel = order[:, :k]
    return sel, softmax(np.take_along_axis(logits, sel, axis=1), axis=1)


def route_permutation(selected: np.ndarray, n_experts: int):
    """Builder-defined segment layout: routes (t, slot)
    stably sorted by expert, tokens ascending inside each expert.

    Returns perm_token (R,), perm_slot (R,), offsets (E+1,), inv (N, k)."""
    n, k = selected.shape
    flat_e = selected.reshape(-1)
    order = np.argsort(flat_e, kind="stable")          # row-major -> t ascending
    counts = np.bincount(flat_e, minlength=n_experts)
    offsets = np.zeros(n_experts + 1, np.int64)
    offsets[1:] = np.cumsum(counts)
    inv = np.empty(n * k, np.int64)
    inv[order] = np.arange(n * k)
    return (order // k).astype(np.int32), (order % k).astype(np.int32), \
        offsets.astype(np.int32), inv.reshape(n, k).astype(np.int32)


def relative_error(got, want) -> float:
    """Frobenius relative error (pipeline.py:349-355)."""
    num = float(np.sqrt(np.sum((np.asarray(got, np.float64) -
                                np.asarray(want, np.float64)) ** 2)))
    den = float(np.sqrt(np.sum(np.asarray(want, np.float64) ** 2)))
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return num / den


def moe_layer(v, w_router, experts, top_k, gemm=lut_gemm, shared=(),
              return_trace=False):
    """The reference fp32 LUT path for one MoE block.

    v: (N, d) fp32 layer input (already rotated when a rotation is online).
    experts: list of (gate, up, down), each (centroids (d_out,G,16) f32,
             ids_packed, g).
    shared: builder-defined always-on experts, weight 1, added after the
            routed sum (not in the reference).
    """
    v = np.ascontiguousarray(v, np.float32)
    n, d = v.shape
    n_exp = len(experts)
    codes, scales = quantize(v, 4)
    router_in = codes.astype(np.float32) * scales[:, None]   # exact (quant.py:8-13)
    logits = matmul_ordered(router_in, np.asarray(w_router, np.float32))
    sel, wts = select_top_k(logits, top_k)
    dense_w = np.zeros((n, n_exp), np.float32)
    np.put_along_axis(dense_w, sel, wts.astype(np.float32), axis=1)
    out = np.zeros((n, d), np.float32)
    f_rows = {}
    for e in range(n_exp):
        rows = np.nonzero((sel == e).any(axis=1))[0]
        if rows.size == 0:
            continue
        (cg, ig, gg), (cu, iu, gu), (cd, idn, gd) = experts[e]
        a = gemm(codes[rows], scales[rows], ig, cg, gg)
        b = gemm(codes[rows], scales[rows], iu, cu, gu)
        h = (silu(a) * b).astype(np.float32)
        hc, hs = quantize(h, 4)
        f = gemm(hc, hs, idn, cd, gd)
        out[rows] = out[rows] + dense_w[rows, e, None] * f
        f_rows[e] = (rows, f)
    for (cg, ig, gg), (cu, iu, gu), (cd, idn, gd) in shared:
        a = gemm(codes, scales, ig, cg, gg)
        b = gemm(codes, scales, iu, cu, gu)
        hc, hs = quantize((silu(a) * b).astype(np.float32), 4)
        out = out + gemm(hc, hs, idn, cd, gd)
    if return_trace:
        return out, dict(codes=codes, scales=scales, logits=logits,
                         selected=sel, weights=wts, f=f_rows)
    return out
