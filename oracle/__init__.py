"""CPU oracle package — TEST INFRASTRUCTURE ONLY (see oracle/oracle.py).

Three layers, all checkers, none of them shipped:
  * `oracle.oracle`   numpy restatement (pinned to tests/golden/*.npz);
  * `cq_*` below      ctypes over oracle/libcq_oracle.so, the C restatement
                      (fast enough for full-size parity checks);
  * `ref_core()`      the reference's own Cython kernel module compiled from
                      /root/reference by oracle/Makefile into oracle/_ref/
                      (travels to the GPU box as a built file).
"""

from __future__ import annotations

import concurrent.futures as _cf
import ctypes
import importlib.util
import os
import subprocess
import sysconfig

import numpy as np

from . import oracle as np_oracle  # noqa: F401  (re-export)
from .oracle import (RngState, build_lut, dense_weight, lut_gemm, matmul_ordered,  # noqa: F401
                     moe_layer, pack_ids, pad_centroids, quantize, reference_gemm,
                     relative_error, route_permutation, select_top_k, silu, softmax,
                     unpack_ids)

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build(ref: bool = True) -> None:
    """Compile the C restatement and, when /root/reference is present, the
    reference's own kernel into oracle/_ref/ (no-op if already built)."""
    targets = ["all"]
    if ref and os.path.exists("/root/reference/pkg/src/codequant/kernels/_core.pyx"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", _HERE, *targets], check=True)


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libcq_oracle.so")
        if not os.path.exists(path):
            build(ref=False)
        lib = ctypes.CDLL(path)
        i64, vp, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        for name in ("cqo_lut_gemm_f32", "cqo_reference_gemm_f32"):
            fn = getattr(lib, name)
            fn.argtypes = [vp, vp, vp, vp, i64, i64, i64, i64, vp, ci]
            fn.restype = ci
        lib.cqo_matmul_f32.argtypes = [vp, vp, vp, i64, i64, i64, ci]
        lib.cqo_quantize_f32.argtypes = [vp, i64, i64, vp, vp]
        _LIB = lib
    return _LIB


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def c_lut_gemm(codes, scales, ids_packed, centroids, g, threads=None, table=True):
    codes = np.ascontiguousarray(codes, np.int8)
    scales = np.ascontiguousarray(scales, np.float32)
    ids_packed = np.ascontiguousarray(ids_packed, np.uint8)
    centroids = np.ascontiguousarray(centroids, np.float32)
    n, d_in = codes.shape
    d_out = centroids.shape[0]
    out = np.zeros((n, d_out), np.float32)
    if n and d_out:
        fn = _lib().cqo_lut_gemm_f32 if table else _lib().cqo_reference_gemm_f32
        rc = fn(_p(codes), _p(scales), _p(ids_packed), _p(centroids), n, d_in, d_out,
                int(g), _p(out), int(threads or os.cpu_count() or 1))
        if rc:
            raise ValueError("oracle gemm: bad group size")
    return out


def c_matmul(a, b, threads=None):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    out = np.empty((a.shape[0], b.shape[1]), np.float32)
    _lib().cqo_matmul_f32(_p(a), _p(b), _p(out), a.shape[0], a.shape[1], b.shape[1],
                          int(threads or os.cpu_count() or 1))
    return out


def c_quantize(x):
    x = np.ascontiguousarray(x, np.float32)
    codes = np.empty(x.shape, np.int8)
    scales = np.empty(x.shape[0], np.float32)
    _lib().cqo_quantize_f32(_p(x), x.shape[0], x.shape[1], _p(codes), _p(scales))
    return codes, scales


def moe_layer_fast(v, w_router, experts, top_k, shared=(), return_trace=False):
    """moe_layer with the C restatement underneath (bitwise identical to the
    numpy path: same quantizer, same ordered chains)."""
    import oracle.oracle as o
    saved = (o.quantize, o.matmul_ordered)
    try:
        o.quantize = lambda x, bits=4: c_quantize(x) if bits == 4 else saved[0](x, bits)
        o.matmul_ordered = c_matmul
        return o.moe_layer(v, w_router, experts, top_k, gemm=c_lut_gemm, shared=shared,
                           return_trace=return_trace)
    finally:
        o.quantize, o.matmul_ordered = saved


# ---------------------------------------------------------------------------
# The reference's own compiled kernel (oracle/_ref), used as the CPU baseline.

_REF = None


def ref_core():
    """Import oracle/_ref/_core*.so (built from the reference's _core.pyx)."""
    global _REF
    if _REF is None:
        path = os.path.join(_HERE, "_ref", "_core" + sysconfig.get_config_var("EXT_SUFFIX"))
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    f"/root/reference is mounted")
        spec = importlib.util.spec_from_file_location("_core", path)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _REF = mod
    return _REF


def ref_lut_gemm(codes, scales, ids_packed, centroids, g, block_tokens=64, threads=1):
    """Restates kernels/compiled.py:27-51: disjoint block-aligned token ranges
    on a thread pool over the reference kernel (GIL released inside)."""
    core = ref_core()
    codes = np.ascontiguousarray(codes, np.int8)
    scales = np.ascontiguousarray(scales, np.float32)
    n = codes.shape[0]
    out = np.zeros((n, centroids.shape[0]), np.float32)
    if n == 0 or centroids.shape[0] == 0:
        return out
    args = (codes, scales, np.ascontiguousarray(ids_packed, np.uint8),
            np.ascontiguousarray(centroids, np.float32), int(g), int(block_tokens))
    if threads <= 1 or n <= block_tokens:
        core.lut_gemm_f32(*args, out, 0, n)
        return out
    n_blocks = -(-n // block_tokens)
    step = -(-n_blocks // threads) * block_tokens
    with _cf.ThreadPoolExecutor(max_workers=threads) as pool:
        futs = [pool.submit(core.lut_gemm_f32, *args, out, t0, min(t0 + step, n))
                for t0 in range(0, n, step)]
        for f in futs:
            f.result()
    return out


def moe_layer_reference(v, w_router, experts, top_k, threads=None, shared=()):
    """The composed MoE block on the reference's native kernels: router logits
    through _core.matmul_f32, expert GEMMs through _core.lut_gemm_f32 with
    threads = cpu count and block_tokens = ceil(n_e / threads)."""
    import oracle.oracle as o
    core = ref_core()
    threads = int(threads or os.cpu_count() or 1)

    def gemm(codes, scales, ids, cent, g):
        bt = max(1, -(-codes.shape[0] // threads))
        return ref_lut_gemm(codes, scales, ids, cent, g, block_tokens=bt, threads=threads)

    def mm(a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        out = np.zeros((a.shape[0], b.shape[1]), np.float32)
        core.matmul_f32(a, b, out)
        return out

    saved = o.matmul_ordered
    try:
        o.matmul_ordered = mm
        return o.moe_layer(v, w_router, experts, top_k, gemm=gemm, shared=shared)
    finally:
        o.matmul_ordered = saved
