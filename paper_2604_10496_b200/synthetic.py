"""Seeded synthetic MoE inputs.

`moe_inputs` draws on the host with the reference's substream scheme
(linalg.RngState, linalg.py:32-53: Philox keyed by SHA-256 of
"seed:tag:index"), so the oracle and the device see the same bytes; the golden
fixtures pin its output digest (tests/golden/make_golden.py).
`moe_inputs_device` draws the same distributions directly on the GPU with a
torch generator — for benchmark-size layers (Mixtral: 1.4 GB of codebooks)
where host generation would dominate; those are checked through
size-independent properties and the GPU ordered path, not the CPU oracle.

Distributions: v ~ N(0,1) rounded to bfloat16 (the device activation dtype)
and handed to the oracle as its exact float32 upcast; router W ~ N(0,1)/sqrt(d);
centroids ~ N(0,1)/sqrt(d_in) float32 per (row, group, k); ids ~ U{0..15}.
"""

from __future__ import annotations

import hashlib

import numpy as np
import torch

from .lutgemm import PackedClusteredWeights


class RngState:
    def __init__(self, seed: int):
        self.seed = int(seed)

    def stream(self, tag: str, index: int = 0) -> np.random.Generator:
        digest = hashlib.sha256(f"{self.seed}:{tag}:{index}".encode()).digest()
        return np.random.Generator(np.random.Philox(key=np.frombuffer(digest[:16], np.uint64)))


def round_bf16(v: np.ndarray) -> np.ndarray:
    """float32 -> nearest-even bfloat16 -> float32 (exact upcast)."""
    bits = v.astype(np.float32).view(np.uint32).astype(np.uint64)
    bits = ((bits + 0x7FFF + ((bits >> 16) & 1)) >> 16) << 16
    return bits.astype(np.uint32).view(np.float32)


def pack_ids_np(ids: np.ndarray) -> np.ndarray:
    if ids.shape[1] % 2:
        ids = np.concatenate([ids, np.zeros((ids.shape[0], 1), np.uint8)], axis=1)
    return (ids[:, 0::2] | (ids[:, 1::2] << np.uint8(4))).astype(np.uint8)


def plant_outliers(v: np.ndarray, channel_scale: float = 8.0, row_scale: float = 50.0) -> np.ndarray:
    """The planted-outlier activation variant (after
    generate_calibration, model.py:191-221): max(1, d/16) evenly spaced channels
    scaled by channel_scale (the pipeline default 8, pipeline.py:59) and max(1,
    n/50) evenly spaced rows by row_scale; bf16-exact again afterwards."""
    v = np.array(v, dtype=np.float32, copy=True)
    n, d = v.shape
    v[:, np.linspace(0, d - 1, max(1, d // 16)).astype(int)] *= channel_scale
    v[np.linspace(0, n - 1, max(1, n // 50)).astype(int)] *= row_scale
    return round_bf16(v)


def moe_inputs_host(seed: int, n: int, d: int, ff: int, n_exp: int, g: int, n_shared: int = 0,
                    outliers: bool = False):
    """Host arrays: v (n,d) f32 (bf16-exact), w_router (d,E) f32, experts =
    [(gate, up, down)] with each site (centroids (d_out, d_in/g, 16) f32,
    ids_packed (d_out, d_in/2) u8, g).  g = 0: embedding-wise groups (g = the
    site's d_in)."""
    rng = RngState(seed)
    v = round_bf16(rng.stream("moe.v").standard_normal((n, d)).astype(np.float32))
    if outliers:
        v = plant_outliers(v)
    w_router = (rng.stream("moe.router").standard_normal((d, n_exp)) / np.sqrt(d)).astype(np.float32)

    def expert(tag):
        mats = []
        for site, (di, do) in (("gate", (d, ff)), ("up", (d, ff)), ("down", (ff, d))):
            gs = g or di
            cents = (rng.stream(f"{tag}.{site}.c").standard_normal((do, di // gs, 16))
                     / np.sqrt(di)).astype(np.float32)
            ids = rng.stream(f"{tag}.{site}.i").integers(0, 16, (do, di)).astype(np.uint8)
            mats.append((cents, pack_ids_np(ids), gs))
        return mats

    experts = [expert(f"moe.e{e}") for e in range(n_exp)]
    shared = [expert(f"moe.s{s}") for s in range(n_shared)]
    return v, w_router, experts, shared


def input_digest(v, w_router, experts) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(v).tobytes())
    h.update(np.ascontiguousarray(w_router).tobytes())
    for mats in experts:
        for cents, ids, _ in mats:
            h.update(np.ascontiguousarray(cents).tobytes())
            h.update(np.ascontiguousarray(ids).tobytes())
    return h.hexdigest()


def to_device_experts(experts):
    """[(gate, up, down)] host tuples -> PackedClusteredWeights triples."""
    out = []
    for mats in experts:
        out.append(tuple(PackedClusteredWeights(torch.from_numpy(c), torch.from_numpy(i), c.shape[1] * g, g)
                         for c, i, g in mats))
    return out


def moe_inputs_device(seed: int, n: int, d: int, ff: int, n_exp: int, g: int, n_shared: int = 0,
                      outliers: bool = False, kc: int = 16):
    """Same distributions drawn on cuda:0 (torch Philox).  Returns v (n,d) bf16,
    w_router (d,E) f32 and stacked sites as dicts of device tensors.  g = 0:
    embedding-wise groups (ExpertStack takes group_size 0 the same way).  kc:
    centroids per group (K; ids < K, centroids zero-padded to 16 as
    pack_weights does, lutgemm.py:109-110)."""
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    v = torch.randn((n, d), generator=gen, device="cuda")
    if outliers:
        v = torch.from_numpy(plant_outliers(v.cpu().numpy())).cuda()
    v = v.to(torch.bfloat16)
    w_router = torch.randn((d, n_exp), generator=gen, device="cuda") / float(np.sqrt(d))

    def stack(ne):
        sites = {}
        for site, (di, do) in (("gate", (d, ff)), ("up", (d, ff)), ("down", (ff, d))):
            cents = torch.randn((ne, do, di // (g or di), 16), generator=gen, device="cuda") / float(np.sqrt(di))
            if kc < 16:
                cents[..., kc:] = 0.0
                lo = torch.randint(0, kc, (ne, do, di // 2), generator=gen, device="cuda", dtype=torch.int32)
                hi = torch.randint(0, kc, (ne, do, di // 2), generator=gen, device="cuda", dtype=torch.int32)
                ids = (lo | (hi << 4)).to(torch.uint8)
            else:
                ids = torch.randint(0, 256, (ne, do, di // 2), generator=gen, device="cuda",
                                    dtype=torch.int32).to(torch.uint8)
            sites[site] = (ids, cents, di, do)
        return sites

    return v, w_router, stack(n_exp), (stack(n_shared) if n_shared else None)
