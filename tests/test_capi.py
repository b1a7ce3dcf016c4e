"""CPU-side checks of the boundary: the C-ABI library loads, exports every
symbol include/cq_b200.h declares, and the host API validates like the
reference (no compute calls without a GPU)."""

import ctypes
import os
import re

import numpy as np
import pytest
import torch

from paper_2604_10496_b200 import _lib
from paper_2604_10496_b200.errors import ConfigError, ShapeError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "cq_b200.h")).read()
    return sorted(set(re.findall(r"CQ_API\s+[\w\s\*]+?\b(cq_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load_library()
    syms = _header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTS)


def test_abi_version_and_counter():
    lib = _lib.load_library()
    assert lib.cq_abi_version() == 6
    assert lib.cq_launch_count() >= 0


def test_workspace_layout_is_aligned_and_monotone():
    lib = _lib.load_library()
    d = _lib.MoEDesc()
    d.d_model, d.d_ff, d.n_experts, d.top_k, d.n_local_experts = 4096, 14336, 8, 2, 8
    offs = (ctypes.c_int64 * len(_lib.WS_NAMES))()
    total = lib.cq_moe_workspace(ctypes.byref(d), 64, offs)
    o = list(offs)
    assert all(x % 256 == 0 for x in o) and o == sorted(o) and total >= o[-1]
    assert o[_lib.WS_NAMES.index("hidden") + 1] - o[_lib.WS_NAMES.index("hidden")] >= 128 * 14336 * 4


def test_status_codes_map_to_reference_errors():
    lib = _lib.load_library()
    # a shape error raised by the library itself (validated before any launch)
    rc = lib.cq_reference_gemm_f32(None, None, None, None, 1, 10, 4, 3, None, None)
    assert rc == _lib.CQ_ERR_SHAPE
    with pytest.raises(ShapeError, match="group size"):
        _lib.check(rc)
    rc = lib.cq_route_topk(None, 4, 4, 5, None, None, None)
    with pytest.raises(ConfigError):
        _lib.check(rc)


def test_no_cpu_fallback():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.lib()


def test_pack_weights_validation_mirrors_reference():
    from paper_2604_10496_b200 import lutgemm
    ids = np.zeros((2, 4), dtype=np.uint8)
    # the reference's messages (lutgemm.py:96-108); these fail before any device use
    with pytest.raises(ShapeError, match="nibble"):
        lutgemm.pack_weights(np.ones((2, 1, 17)), ids, 4)
    with pytest.raises(ShapeError, match="out of centroid range"):
        lutgemm.pack_weights(np.ones((2, 1, 3)), np.full((2, 4), 3, dtype=np.uint8), 4)
    with pytest.raises(ShapeError, match="does not match"):
        lutgemm.pack_weights(np.ones((2, 2, 3)), ids, 4)
    with pytest.raises(ShapeError):
        lutgemm.build_lut(np.zeros(5))


def test_build_lut_is_one_float_multiply():
    from paper_2604_10496_b200 import build_lut
    cents = np.random.default_rng(3).standard_normal(16).astype(np.float32)
    t = build_lut(cents)
    for c in range(16):
        for code in range(-8, 8):
            assert t.entry(c, code) == np.float32(cents[c]) * np.float32(code)


def test_quant_spec_and_nibbles():
    from paper_2604_10496_b200.quant import QuantSpec, pack_nibbles, unpack_nibbles
    with pytest.raises(ShapeError):
        QuantSpec(5)
    assert pack_nibbles(np.array([1, 2], np.uint8)) == b"\x21"
    assert pack_nibbles(np.array([15], np.uint8)) == b"\x0f"
    for value in range(256):
        assert pack_nibbles(unpack_nibbles(bytes([value]), 2)) == bytes([value])
    with pytest.raises(ShapeError):
        unpack_nibbles(b"\x00", 3)
