"""Activation quantization on the device (reference quant.py:24-157).

`quantize_activations` keeps the reference's name, arguments and errors; the
work runs in `cq_quantize_a4` (bit-exact with quant.py:89-100 on float32
input).  Tensors are torch CUDA tensors.  The nibble codecs stay on the host:
they are the container byte format (quant.py:140-157), not the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, DivergenceError, ShapeError

_ALLOWED_BITS = (2, 3, 4, 8)


@dataclass(frozen=True)
class QuantSpec:
    """Bit width plus grouping (quant.py:24-47)."""

    bits: int
    group_size: int | None = None

    def __post_init__(self):
        if self.bits not in _ALLOWED_BITS:
            raise ShapeError(f"bits must be one of {_ALLOWED_BITS}, got {self.bits}")
        if self.group_size is not None and self.group_size < 1:
            raise ShapeError(f"group_size must be positive, got {self.group_size}")

    @property
    def qmax(self) -> int:
        return 2 ** (self.bits - 1) - 1

    @property
    def qmin(self) -> int:
        return -(2 ** (self.bits - 1))


@dataclass
class QuantizedActivations:
    """codes: int8 (N, d) CUDA tensor; scales: float32 (N,) CUDA tensor."""

    codes: torch.Tensor
    scales: torch.Tensor
    bits: int


def _as_device(x, dtype=None) -> torch.Tensor:
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(x)
    if dtype is not None and x.dtype != dtype:
        x = x.to(dtype)
    return x.to("cuda", non_blocking=True).contiguous()


def quantize_activations(x, spec: QuantSpec = QuantSpec(4), check_finite: bool = True
                         ) -> QuantizedActivations:
    """Per-token symmetric quantization with snapped scales (quant.py:89-100).

    x: (N, d) float32 or bfloat16 (CUDA tensor or host array, copied to the
    device).  Raises DivergenceError on non-finite input like the reference
    (the kernel sets a device flag; reading it is one host sync);
    `check_finite=False` skips that read on the hot path.
    """
    if spec.bits != 4:
        raise ConfigError(f"device quantizer takes 4-bit codes, got {spec.bits}-bit")
    if isinstance(x, np.ndarray) and x.dtype == np.float64:
        raise ShapeError("device quantizer takes float32/bfloat16 activations")
    x = _as_device(x)
    if x.dim() != 2:
        raise ShapeError(f"activations must be 2-D, got shape {tuple(x.shape)}")
    n, d = x.shape
    codes = torch.empty((n, d), dtype=torch.int8, device=x.device)
    scales = torch.empty((n,), dtype=torch.float32, device=x.device)
    if n:
        flag = torch.zeros(1, dtype=torch.int32, device=x.device) if check_finite else None
        _lib.check(_lib.lib().cq_quantize_a4(x.data_ptr(), _lib.dtype_code(x), n, d,
                                             codes.data_ptr(), scales.data_ptr(), _lib.ptr(flag),
                                             _lib.stream()))
        if check_finite and int(flag.item()):
            raise DivergenceError("non-finite activation input to quantizer")
    return QuantizedActivations(codes, scales, spec.bits)


def dequantize(qa: QuantizedActivations) -> torch.Tensor:
    return qa.codes.float() * qa.scales[:, None]


def fake_quant(x, spec: QuantSpec = QuantSpec(4)) -> torch.Tensor:
    """Q(.): quantize then dequantize (quant.py:103-109)."""
    return dequantize(quantize_activations(x, spec))


def pack_nibbles(ids) -> bytes:
    """Two 4-bit ids per byte, low nibble first; odd length pads with 0."""
    flat = np.ascontiguousarray(ids, dtype=np.uint8).reshape(-1)
    if flat.size and flat.max() > 15:
        raise ShapeError("nibble values must be in 0..15")
    if flat.size % 2:
        flat = np.concatenate([flat, np.zeros(1, np.uint8)])
    return (flat[0::2] | (flat[1::2] << np.uint8(4))).tobytes()


def unpack_nibbles(data: bytes, count: int) -> np.ndarray:
    raw = np.frombuffer(data, dtype=np.uint8)
    if count > 2 * raw.size:
        raise ShapeError(f"need {count} nibbles but have {2 * raw.size}")
    out = np.empty(raw.size * 2, np.uint8)
    out[0::2] = raw & np.uint8(0x0F)
    out[1::2] = raw >> np.uint8(4)
    return out[:count]
