"""The reference-side drop-in module (integration/codequant_b200_backend.py)
against the reference's own kernel registry (kernels/__init__.py:19-94), on
CPU: it installs as a backend, exposes the module contract of the compiled /
numpy backends with the same signatures, and refuses to run without a GPU
(no CPU fallback).  Runs where /root/reference is mounted (this container);
the GPU-side bytewise checks are tests/test_gpu_integration.py."""

import importlib
import inspect
import os
import sys

import numpy as np
import pytest
import torch

from integration import codequant_b200_backend as b200

REF_SRC = "/root/reference/pkg/src"


@pytest.fixture()
def ref_kernels(monkeypatch):
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference not mounted")
    monkeypatch.setenv("CODEQUANT_BACKEND", "python")
    monkeypatch.syspath_prepend(REF_SRC)
    for name in [m for m in sys.modules if m == "codequant" or m.startswith("codequant.")]:
        monkeypatch.delitem(sys.modules, name)
    kernels = importlib.import_module("codequant.kernels")
    monkeypatch.setattr(kernels, "_BACKENDS", dict(kernels._BACKENDS))
    monkeypatch.setattr(kernels, "_ALIASES", dict(kernels._ALIASES))
    return kernels


def test_installs_into_the_reference_registry(ref_kernels):
    b200.install(ref_kernels)
    assert ref_kernels.get_backend("b200") is b200
    assert ref_kernels.get_backend("cuda") is b200
    assert "b200" in ref_kernels.available_backends()


def test_module_contract_matches_the_reference_backends(ref_kernels):
    fallback = importlib.import_module("codequant.kernels.fallback")
    for fn in ("matmul_f32", "matmul_f64", "lut_gemm_f32", "reference_gemm_f32"):
        assert inspect.signature(getattr(b200, fn)) == inspect.signature(getattr(fallback, fn)), fn
    assert isinstance(b200.NAME, str)


def test_matmul_f64_is_the_reference_host_loop(ref_kernels):
    fallback = importlib.import_module("codequant.kernels.fallback")
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal((5, 7)), rng.standard_normal((7, 3))
    want, got = np.zeros((5, 3)), np.zeros((5, 3))
    fallback.matmul_f64(a, b, want)
    b200.matmul_f64(a, b, got)
    assert got.tobytes() == want.tobytes()


def test_no_cpu_fallback():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    q = np.zeros((1, 16), np.int8)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        b200.lut_gemm_f32(q, np.ones(1, np.float32), np.zeros((8, 8), np.uint8), np.zeros((8, 1, 16), np.float32),
                          16)
