"""Expert-parallel protocol on CPU: world_size 2 and 4 over gloo, the CPU oracle
as the compute backend (ep.EPMoE: counts-first all_to_all-v of packed-nibble
rows, receiver-side partial sums, source-side combine, replicated shared
experts).  The exact-row protocol must reproduce the single-process
reference composition bit for bit (same per-route arithmetic, ascending-expert
combine); the dedup protocol within fp32 re-association of the cross-rank adds,
and bit for bit at world 1."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as o
from paper_2604_10496_b200.ep import (EPMoE, expert_range, header_bytes, pack_rows, plan_rows,
                                      unpack_rows)
from paper_2604_10496_b200.synthetic import moe_inputs_host


class OracleBackend:
    """Test-only compute backend over the numpy oracle (CPU tensors)."""

    def __init__(self, w_router, experts_local, k, shared=()):
        self.w = np.asarray(w_router, np.float32)
        self.local, self.k, self.sh = experts_local, k, shared

    def route(self, x):
        codes, scales = o.quantize(x.numpy().astype(np.float32), 4)
        logits = o.matmul_ordered(codes.astype(np.float32) * scales[:, None], self.w)
        sel, wts = o.select_top_k(logits, self.k)
        return (torch.from_numpy(codes), torch.from_numpy(scales), torch.from_numpy(sel.astype(np.int64)),
                torch.from_numpy(wts.astype(np.float32)))

    @staticmethod
    def _ffn(mats, codes, scales):
        (cg, ig, gg), (cu, iu, gu), (cd, idn, gd) = mats
        a = o.lut_gemm(codes, scales, ig, cg, gg)
        b = o.lut_gemm(codes, scales, iu, cu, gu)
        hc, hs = o.quantize((o.silu(a) * b).astype(np.float32), 4)
        return o.lut_gemm(hc, hs, idn, cd, gd)

    def experts(self, codes, scales, eid, n_local):
        codes, scales, eid = codes.numpy(), scales.numpy(), eid.numpy()
        d = self.local[0][2][0].shape[0]
        out = np.zeros((codes.shape[0], d), np.float32)
        for e in range(n_local):
            rows = np.nonzero(eid == e)[0]
            if rows.size:
                out[rows] = self._ffn(self.local[e], codes[rows], scales[rows])
        return torch.from_numpy(out)

    def shared(self, codes, scales):
        if not self.sh:
            return None
        return [torch.from_numpy(self._ffn(m, codes.numpy(), scales.numpy())) for m in self.sh]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, dedup, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seed, n, d, ff, E, k, g, n_sh = cfg
        v, w, experts, shared = moe_inputs_host(seed, n, d, ff, E, g, n_shared=n_sh)
        begin, per = expert_range(E, world, rank)
        be = OracleBackend(w, experts[begin:begin + per], k, shared)
        layer = EPMoE(be, E, k, rank, world, dedup=dedup)
        lo, hi = rank * n // world, (rank + 1) * n // world
        out = layer(torch.from_numpy(v[lo:hi]))
        result_q.put((rank, (out.numpy(), layer.last)))
    except Exception as exc:  # surface the failure instead of a queue timeout
        result_q.put((rank, repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


def _run(world, cfg, dedup):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, dedup, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = dict(q.get(timeout=180) for _ in range(world))
    for r in range(world):
        assert not isinstance(parts[r], str), parts[r]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return np.concatenate([parts[r][0] for r in range(world)]), [parts[r][1] for r in range(world)]


CFGS = [(3, 24, 64, 96, 4, 2, 32, 0), (7, 17, 128, 64, 6, 3, 64, 0), (11, 20, 64, 64, 8, 3, 32, 2)]


@pytest.mark.parametrize("cfg", CFGS)
def test_ep_exact_rows_world2_bitwise_equal_oracle(cfg):
    seed, n, d, ff, E, k, g, n_sh = cfg
    got, _ = _run(2, cfg, dedup=False)
    v, w, experts, shared = moe_inputs_host(seed, n, d, ff, E, g, n_shared=n_sh)
    want = o.moe_layer(v, w, experts, k, shared=shared)
    assert np.array_equal(got.view(np.int32), want.view(np.int32))


@pytest.mark.parametrize("world", [2, 4])
def test_ep_dedup_rows_shared_experts_match_oracle(world):
    """DS-shaped (shared experts, top-k spread over ranks): the dedup protocol
    sends one row per (token, peer) — fewer rows than routes — and agrees with
    the oracle to fp32 re-association."""
    cfg = (13, 24, 64, 64, 8, 3, 32, 2)
    seed, n, d, ff, E, k, g, n_sh = cfg
    got, stats = _run(world, cfg, dedup=True)
    v, w, experts, shared = moe_inputs_host(seed, n, d, ff, E, g, n_shared=n_sh)
    want = o.moe_layer(v, w, experts, k, shared=shared)
    assert o.relative_error(got, want) <= 1e-6
    rows, routes = sum(s["send_rows"] for s in stats), sum(s["routes"] for s in stats)
    assert routes == n * k and rows < routes


def test_ep_dedup_world1_bitwise():
    """At world 1 every token's experts share the rank: the dedup protocol is
    the single-GPU composition bit for bit (exchanges are identity copies)."""
    seed, n, d, ff, E, k, g, n_sh = 5, 16, 64, 64, 4, 2, 32, 1
    v, w, experts, shared = moe_inputs_host(seed, n, d, ff, E, g, n_shared=n_sh)

    def ident(out, inp, os_, is_):
        out.copy_(inp)

    layer = EPMoE(OracleBackend(w, experts, k, shared), E, k, 0, 1, dedup=True, exchange=ident)
    got = layer(torch.from_numpy(v)).numpy()
    want = o.moe_layer(v, w, experts, k, shared=shared)
    assert np.array_equal(got.view(np.int32), want.view(np.int32))


@pytest.mark.parametrize("dedup", [True, False])
@pytest.mark.parametrize("d", [64, 48])
def test_row_protocol_round_trip(dedup, d):
    """plan_rows / pack_rows / unpack_rows: codes (packed nibbles at d % 32 == 0,
    int8 otherwise), scales, routes and weights survive the row format; rows
    are ordered by peer then token; every route appears once; src_slot points
    each token at its rows in ascending peer (dedup) / expert order."""
    rng = np.random.default_rng(3)
    n, E, world, k = 37, 16, 4, 5
    per = E // world
    sel = torch.from_numpy(np.stack([rng.permutation(E)[:k] for _ in range(n)]))
    wts = torch.from_numpy(rng.random((n, k)).astype(np.float32))
    codes = torch.from_numpy(rng.integers(-8, 8, (n, d)).astype(np.int8))
    scales = torch.from_numpy(rng.random(n).astype(np.float32))
    p = plan_rows(sel, wts, E, world, dedup)
    rows = pack_rows(codes, scales, p)
    cb = d // 2 if d % 32 == 0 else d
    assert rows.shape == (p.tok.numel(), cb + header_bytes(p.kr))
    rc, rs, rm, re, rw = unpack_rows(rows, d, p.kr)
    assert torch.equal(rc, codes[p.tok]) and torch.equal(rs, scales[p.tok])
    assert torch.equal(rm, p.m) and torch.equal(re, p.e) and torch.equal(rw, p.w)
    assert (torch.diff(p.dest) >= 0).all()
    for g in range(world):
        assert (torch.diff(p.tok[p.dest == g]) > 0).all() if dedup else (torch.diff(p.tok[p.dest == g]) >= 0).all()
    assert int(p.counts.sum()) == rows.shape[0] and int(p.routes.sum()) == n * k
    # every (token, expert) route exactly once, with its weight
    got = {}
    for r in range(rows.shape[0]):
        for j in range(int(rm[r])):
            got[(int(p.tok[r]), int(p.dest[r]) * per + int(re[r, j]))] = float(rw[r, j])
    assert len(got) == n * k
    for t in range(n):
        for s in range(k):
            assert got[(t, int(sel[t, s]))] == (float(wts[t, s]) if dedup else 1.0)
        slots = p.src_slot[t][p.src_slot[t] >= 0].long()
        assert torch.equal(p.tok[slots], torch.full_like(slots, t))
        keys = p.dest[slots] if dedup else p.dest[slots] * per + re[slots, 0]
        assert (torch.diff(keys) > 0).all()
