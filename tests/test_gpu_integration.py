"""Acceptance criterion #8 of the reference (tests/test_acceptance.py:358-387)
through the reference-side backend module (integration/codequant_b200_backend.py):
the 216 instances are regenerated with the reference test's own numpy draws,
and the backend's lut_gemm_f32 and reference_gemm_f32 must produce the exact
bytes the reference produced (SHA-256 recorded by tests/golden/make_golden.py
from the reference itself), for every (block_tokens, threads) variant."""

import hashlib
from itertools import product

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from integration import codequant_b200_backend as b200  # noqa: E402
from oracle import oracle as o  # noqa: E402


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _instances():
    """tests/test_acceptance.py:361-373, draw for draw."""
    combos = [(n, d, g) for n, d in product((1, 7, 64, 256), (16, 64, 256)) for g in sorted({16, 64, d}) if g <= d]
    instances = 0
    for seed in range(9):
        for n_tokens, d_in, g in combos:
            rng = np.random.default_rng(1_000_003 * seed + 1009 * n_tokens + 13 * d_in + g)
            d_out = 16 if instances % 2 else 8
            k = 16 if instances % 3 else 5
            x = rng.standard_normal((n_tokens, d_in))
            if instances % 3 == 0:
                x[: max(1, n_tokens // 4)] = 0.0
            centroids = rng.standard_normal((d_out, d_in // g, k)).astype(np.float32)
            ids = rng.integers(0, k, (d_out, d_in), dtype=np.uint8)
            yield (seed, n_tokens, d_in, g, d_out, k), x, centroids, ids
            instances += 1


def test_acceptance8_bytes_through_the_backend_module(golden):
    gold = golden("acceptance8.npz")
    n_inst = 0
    for i, (p, x, centroids, ids) in enumerate(_instances()):
        assert tuple(gold["params"][i]) == p
        codes, scales = o.quantize(x, 4)          # the reference's quantizer (fp64 in), pinned by quant.npz
        scales32 = scales.astype(np.float32)      # lutgemm.py:126
        assert _sha(codes) == str(gold["codes_sha"][i]) and _sha(scales32) == str(gold["scales_sha"][i])
        seed, n_tokens, d_in, g, d_out, k = p
        cent16 = o.pad_centroids(centroids)       # pack_weights (lutgemm.py:109-116)
        packed = o.pack_ids(ids)
        want = b200.reference_gemm_f32(codes, scales32, packed, cent16, g)
        assert _sha(want) == str(gold["out_sha"][i]), p
        for bt, th in ((64, 1), (1, 1), (17, 1), (4096, 1), (64, 3)):
            got = b200.lut_gemm_f32(codes, scales32, packed, cent16, g, block_tokens=bt, threads=th)
            assert got.tobytes() == want.tobytes(), (p, bt, th)
        n_inst += 1
    assert n_inst == len(gold["params"]) >= 200


def test_matmul_f32_bitwise_ordered_chain():
    import oracle
    rng = np.random.default_rng(5)
    for m, k, n in ((1, 1, 1), (7, 300, 9), (64, 1024, 8), (33, 2048, 128), (5, 0, 3)):
        a = rng.standard_normal((m, k)).astype(np.float32)
        b = rng.standard_normal((k, n)).astype(np.float32)
        out = np.zeros((m, n), np.float32)
        b200.matmul_f32(a, b, out)
        want = oracle.c_matmul(a, b) if k else np.zeros((m, n), np.float32)
        assert out.tobytes() == want.tobytes(), (m, k, n)
