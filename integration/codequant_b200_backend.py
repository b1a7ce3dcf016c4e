"""CodeQuant kernel backend on a B200 — the reference-side drop-in module.

A maintainer copies this file to `pkg/src/codequant/kernels/b200.py` and adds
two lines to the registry (`kernels/__init__.py:19-35`):

    from . import b200 as _b200            # OSError / RuntimeError: no library or GPU
    _BACKENDS["b200"] = _b200; _ALIASES.update(b200="b200", cuda="b200")

after which `CODEQUANT_BACKEND=b200` (or `get_backend("b200")`) routes the
reference's `lut_gemm`, `reference_gemm` and float32 `linalg.matmul` through
libcq_b200.so.  Same module contract as `kernels/compiled.py:16-61` and
`kernels/fallback.py:14-80`: `NAME`, `matmul_f32/f64(a, b, out)`,
`lut_gemm_f32(q, scales, ids_packed, centroids, g, block_tokens=64, threads=1)`,
`reference_gemm_f32(...)`, host numpy arrays in and out.

Arithmetic contract (the registry's, kernels/__init__.py:1-9): bitwise
interchangeable with the compiled and numpy backends.  `lut_gemm_f32` and
`reference_gemm_f32` both run the ordered chain kernel (csrc/ordered.cu), so
`lut_gemm(...).tobytes() == reference_gemm(...).tobytes()` holds as acceptance
#8 asserts (tests/test_acceptance.py:358-387); `block_tokens` / `threads` never
change a result (one writer per output, kernels/compiled.py:1-6).  float64
matmul is calibration-only (outside the Stage-4 path) and stays on the host.

The C ABI (include/cq_b200.h) takes plain device pointers; torch only supplies
device memory and the stream.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

NAME = "b200"

_HERE = os.path.dirname(os.path.abspath(__file__))
_DEFAULT_LIB = os.path.join(os.path.dirname(_HERE), "paper_2604_10496_b200", "libcq_b200.so")
_LIB = None
_vp, _i64 = ctypes.c_void_p, ctypes.c_int64


def _lib():
    """libcq_b200.so (CQ_B200_LIB overrides the path) — raises without a GPU:
    this backend has no CPU fallback."""
    global _LIB
    if _LIB is None:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("the b200 kernel backend needs a CUDA device; there is no CPU fallback")
        lib = ctypes.CDLL(os.environ.get("CQ_B200_LIB", _DEFAULT_LIB))
        for fn in ("cq_lut_gemm_f32", "cq_reference_gemm_f32"):
            getattr(lib, fn).argtypes = [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp]
            getattr(lib, fn).restype = ctypes.c_int
        lib.cq_matmul_f32.argtypes = [_vp, _vp, _vp, _i64, _i64, _i64, _vp]
        lib.cq_matmul_f32.restype = ctypes.c_int
        lib.cq_last_error.restype = ctypes.c_char_p
        _LIB = lib
    return _LIB


def _errors():
    try:  # inside the reference package
        from ..errors import ConfigError, DivergenceError, ShapeError  # type: ignore
    except (ImportError, ValueError):
        from paper_2604_10496_b200.errors import ConfigError, DivergenceError, ShapeError
    return ShapeError, ConfigError, DivergenceError


def _check(rc: int) -> None:
    if rc:
        shape, config, diverge = _errors()
        msg = _lib().cq_last_error().decode(errors="replace")
        raise {1: shape, 2: config, 3: diverge, 5: config}.get(rc, RuntimeError)(msg)


def _dev(a, dtype):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).cuda()


def _stream() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream


def _gemm(fn, q, scales, ids_packed, centroids, g):
    import torch
    n, d_in = q.shape
    d_out = centroids.shape[0]
    if n == 0 or d_out == 0:
        return np.zeros((n, d_out), dtype=np.float32)
    dq, ds = _dev(q, np.int8), _dev(scales, np.float32)
    di, dc = _dev(ids_packed, np.uint8), _dev(centroids, np.float32)
    out = torch.empty((n, d_out), dtype=torch.float32, device="cuda")
    _check(fn(dq.data_ptr(), ds.data_ptr(), di.data_ptr(), dc.data_ptr(), n, d_in, d_out, int(g), out.data_ptr(),
              _stream()))
    return out.cpu().numpy()


def lut_gemm_f32(q, scales, ids_packed, centroids, g, block_tokens=64, threads=1):
    return _gemm(_lib().cq_lut_gemm_f32, q, scales, ids_packed, centroids, g)


def reference_gemm_f32(q, scales, ids_packed, centroids, g, block_tokens=64, threads=1):
    return _gemm(_lib().cq_reference_gemm_f32, q, scales, ids_packed, centroids, g)


def matmul_f32(a, b, out):
    """out (zeroed by the caller, kernels/__init__.py:66-69) = a @ b, k ascending."""
    import torch
    m, k = a.shape
    n = b.shape[1]
    if m * n == 0:
        return
    da, db = _dev(a, np.float32), _dev(b, np.float32)
    o = torch.empty((m, n), dtype=torch.float32, device="cuda")
    _check(_lib().cq_matmul_f32(da.data_ptr(), db.data_ptr(), o.data_ptr(), m, k, n, _stream()))
    out[...] = o.cpu().numpy()


def matmul_f64(a, b, out):
    """float64 is calibration arithmetic (outside the Stage-4 path): the host
    ordered loop, as kernels/fallback.py:14-27."""
    kdim = a.shape[1]
    if kdim == 0 or out.size == 0:
        return
    tmp = np.empty_like(out)
    for kk in range(kdim):
        np.multiply(a[:, kk, None], b[kk, None, :], out=tmp)
        np.add(out, tmp, out=out)


def install(kernels_module) -> None:
    """The registry lines of INTEGRATION.md, applied to an imported
    `codequant.kernels` module (in memory; used by the tests)."""
    import sys
    kernels_module._BACKENDS[NAME] = sys.modules[__name__]
    kernels_module._ALIASES.update({"b200": "b200", "cuda": "b200"})
