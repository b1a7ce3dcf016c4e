"""Backend registry with the reference's interface (kernels/__init__.py:19-94).

The reference selects between a compiled and a numpy backend; this package
has exactly one backend, ``"b200"`` (libcq_b200.so on an sm_100a device).
There is no dispatch and no fallback: asking for anything else raises, and so
does any call without a CUDA device.  Arrays are CUDA tensors.
"""

from __future__ import annotations

import os

import torch

from . import _lib

NAME = "b200"
_ALIASES = {"b200": "b200", "cuda": "b200", "sm100a": "b200"}


def available_backends() -> tuple[str, ...]:
    return (NAME,)


def get_backend(name: str):
    key = _ALIASES.get(name.lower())
    if key is None:
        raise ValueError(f"unknown kernel backend {name!r}; available: {NAME}")
    import sys
    return sys.modules[__name__]


def _select():
    requested = os.environ.get("CODEQUANT_BACKEND", "").strip()
    return get_backend(requested) if requested else get_backend(NAME)


def active_backend():
    return _select()


def backend_name() -> str:
    return NAME


def matmul_into(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor) -> None:
    """out = a @ b, k ascending, one rounding per op (kernels/__init__.py:72-78)."""
    if a.dtype != torch.float32:
        raise ValueError("device matmul is float32 only (float64 belongs to calibration)")
    _lib.check(_lib.lib().cq_matmul_f32(a.data_ptr(), b.data_ptr(), out.data_ptr(), a.shape[0],
                                        a.shape[1], b.shape[1], _lib.stream()))


def unpack_ids(ids_packed: torch.Tensor, d_in: int) -> torch.Tensor:
    out = torch.empty((ids_packed.shape[0], d_in), dtype=torch.uint8, device=ids_packed.device)
    _lib.check(_lib.lib().cq_unpack_ids(ids_packed.data_ptr(), ids_packed.shape[0], d_in,
                                        out.data_ptr(), _lib.stream()))
    return out


def _gemm(fn, q, scales, ids_packed, centroids, g):
    n, d_in = q.shape
    out = torch.empty((n, centroids.shape[0]), dtype=torch.float32, device=q.device)
    if n == 0 or centroids.shape[0] == 0:
        return out.zero_()
    _lib.check(fn(q.data_ptr(), scales.data_ptr(), ids_packed.data_ptr(), centroids.data_ptr(), n,
                  d_in, centroids.shape[0], int(g), out.data_ptr(), _lib.stream()))
    return out


def lut_gemm_f32(q, scales, ids_packed, centroids, g, block_tokens=64, threads=1):
    return _gemm(_lib.lib().cq_lut_gemm_f32, q, scales, ids_packed, centroids, g)


def reference_gemm_f32(q, scales, ids_packed, centroids, g, block_tokens=64, threads=1):
    return _gemm(_lib.lib().cq_reference_gemm_f32, q, scales, ids_packed, centroids, g)
