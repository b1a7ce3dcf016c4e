"""ctypes binding of libcq_b200.so (the C ABI in include/cq_b200.h).

The library is built in-tree by `__graft_entry__.build()` (nvcc, sm_100a).  It
is the only compute backend: if it is missing, or no CUDA device is present,
every entry point raises — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

import torch

from .errors import ConfigError, DivergenceError, ShapeError

_HERE = os.path.dirname(os.path.abspath(__file__))
# CQ_B200_LIB: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("CQ_B200_LIB") or os.path.join(_HERE, "libcq_b200.so")

CQ_OK, CQ_ERR_SHAPE, CQ_ERR_CONFIG, CQ_ERR_DIVERGENCE, CQ_ERR_CUDA, CQ_ERR_UNSUPPORTED = range(6)
CQ_DTYPE_F32, CQ_DTYPE_BF16 = 0, 1
CQ_PATH_AUTO, CQ_PATH_F32, CQ_PATH_TC, CQ_PATH_ORDERED = 0, 1, 2, 3
CQ_TC_UMMA128U, CQ_TC_UMMA128U8 = 2, 3
TC_LAYOUTS = {"umma128u": CQ_TC_UMMA128U, "umma128u8": CQ_TC_UMMA128U8}
WS_NAMES = ("codes", "scales", "logits", "selected", "weights", "counts", "offsets",
            "perm_token", "perm_slot", "inv", "codes_perm", "scales_perm", "hidden",
            "hcodes", "hscales", "fout", "rotated", "shared", "codes_frag", "hcodes_frag", "rot_act",
            "tok_sums", "status", "sh_offsets")

_vp, _i64, _i32, _int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int


class ExpertSite(ctypes.Structure):
    _fields_ = [("ids", _vp), ("centroids", _vp), ("group_size", _i64),
                ("tc_ids", _vp), ("tc_lut", _vp), ("tc_rowscale", _vp), ("tc_planes", _i64),
                ("tc_layout", _i64)]


class MoEDesc(ctypes.Structure):
    _fields_ = [("d_model", _i64), ("d_ff", _i64), ("n_experts", _i64), ("top_k", _i64),
                ("n_local_experts", _i64), ("expert_begin", _i64),
                ("w_router", _vp), ("rotation", _vp),
                ("gate", ExpertSite), ("up", ExpertSite), ("down", ExpertSite),
                ("n_shared", _i64),
                ("sh_gate", ExpertSite), ("sh_up", ExpertSite), ("sh_down", ExpertSite),
                ("path", _i32), ("rotation_tc", _vp), ("flags", _i64)]


FLAG_KEEP_HIDDEN = 1  # CQ_FLAG_KEEP_HIDDEN
FLAG_SELECT_ONLY = 2  # CQ_FLAG_SELECT_ONLY
FLAG_SHARED_MERGED = 4  # CQ_FLAG_SHARED_MERGED


_SIGS = {
    "cq_quantize_a4": [_vp, _int, _i64, _i64, _vp, _vp, _vp, _vp],
    "cq_unpack_ids": [_vp, _i64, _i64, _vp, _vp],
    "cq_reference_gemm_f32": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp],
    "cq_lut_gemm_f32": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp],
    "cq_matmul_f32": [_vp, _vp, _vp, _i64, _i64, _i64, _vp],
    "cq_route_topk": [_vp, _i64, _i64, _i64, _vp, _vp, _vp],
    "cq_moe_forward": [ctypes.POINTER(MoEDesc), _vp, _int, _i64, _vp, _vp, _i64, _vp],
    "cq_moe_route": [ctypes.POINTER(MoEDesc), _vp, _int, _i64, _vp, _i64, _vp],
    "cq_moe_experts": [ctypes.POINTER(MoEDesc), _vp, _vp, _vp, _i64, _vp, _vp, _i64, _vp],
    "cq_moe_combine": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _i64, _vp, _vp],
    "cq_moe_shared_experts": [ctypes.POINTER(MoEDesc), _i64, _vp, _vp, _i64, _vp],
    "cq_moe_profile_experts": [ctypes.POINTER(MoEDesc), _vp, _vp, _vp, _i64, _vp, _vp, _i64, _i32, _vp, _vp],
    "cq_lut8_prepare": [_vp, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp],
    "cq_lut_gemm_tc": [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _i64, _vp],
    "cq_ep_dispatch": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i32, _i32, _i64, _vp, _vp, _i64, _vp, _vp,
                       _vp, _vp],
    "cq_ep_group": [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp],
    "cq_ep_partial": [_vp, _vp, _vp, _i64, _i64, _i64, _i32, _vp, _vp],
    "cq_ep_combine": [_vp, _vp, _vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _vp],
    "cq_rotation_prepare": [_vp, _i64, _vp, _vp],
}

EXPORTS = tuple(_SIGS) + ("cq_last_error", "cq_abi_version", "cq_launch_count", "cq_moe_workspace",
                          "cq_ep_row_bytes", "cq_ep_scratch_bytes", "cq_rotation_prepared_bytes",
                          "cq_lut_gemm_tc_workspace")

_LIB = None


def load_library() -> ctypes.CDLL:
    """Load libcq_b200.so (no device needed)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                               f"(nvcc, sm_100a). There is no CPU fallback.")
        lib = ctypes.CDLL(LIB_PATH)
        for name, argtypes in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = _int
        lib.cq_last_error.restype = ctypes.c_char_p
        lib.cq_abi_version.restype = _int
        lib.cq_launch_count.restype = _i64
        lib.cq_moe_workspace.argtypes = [ctypes.POINTER(MoEDesc), _i64, ctypes.POINTER(_i64)]
        lib.cq_moe_workspace.restype = _i64
        lib.cq_ep_row_bytes.argtypes = [_i64, _i64]
        lib.cq_ep_row_bytes.restype = _i64
        lib.cq_ep_scratch_bytes.argtypes = [_i64, _i64, _i64, _i64, _i64]
        lib.cq_ep_scratch_bytes.restype = _i64
        lib.cq_rotation_prepared_bytes.argtypes = [_i64]
        lib.cq_rotation_prepared_bytes.restype = _i64
        lib.cq_lut_gemm_tc_workspace.argtypes = [_i64, _i64]
        lib.cq_lut_gemm_tc_workspace.restype = _i64
        _LIB = lib
    return _LIB


def lib() -> ctypes.CDLL:
    """The library, after checking a CUDA device is present."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2604_10496_b200 needs a CUDA (B200, sm_100a) device; "
                           "there is no CPU fallback")
    return load_library()


def check(status: int) -> None:
    if status == CQ_OK:
        return
    msg = load_library().cq_last_error().decode(errors="replace")
    if status == CQ_ERR_SHAPE:
        raise ShapeError(msg)
    if status in (CQ_ERR_CONFIG, CQ_ERR_UNSUPPORTED):
        raise ConfigError(msg)
    if status == CQ_ERR_DIVERGENCE:
        raise DivergenceError(msg)
    raise RuntimeError(f"cq_b200 CUDA error: {msg}")


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


_SCRATCH = {}


def scratch(nbytes: int, tag: str = "tc") -> torch.Tensor:
    """A cached device scratch buffer of at least nbytes per (tag, device):
    C entry points take caller-owned workspaces instead of allocating."""
    key = (tag, torch.cuda.current_device())
    buf = _SCRATCH.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device="cuda")
        _SCRATCH[key] = buf
    return buf


def launch_count() -> int:
    return int(load_library().cq_launch_count())


def dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return CQ_DTYPE_F32
    if t.dtype == torch.bfloat16:
        return CQ_DTYPE_BF16
    raise ShapeError(f"activations must be float32 or bfloat16, got {t.dtype}")
