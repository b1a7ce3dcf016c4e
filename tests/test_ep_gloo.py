"""Expert-parallel host logic on CPU: world_size 2 over gloo, the CPU oracle as
the compute backend.  The EP layer must reproduce the single-process reference
composition bit for bit (same per-route arithmetic, same ascending-expert
combine)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as o
from paper_2604_10496_b200.ep import EPMoE, expert_range, plan_dispatch
from paper_2604_10496_b200.synthetic import moe_inputs_host


class OracleBackend:
    """Test-only compute backend over the numpy oracle (CPU tensors)."""

    def __init__(self, w_router, experts_local):
        self.w = np.asarray(w_router, np.float32)
        self.local = experts_local

    def route(self, x):
        codes, scales = o.quantize(x.numpy().astype(np.float32), 4)
        logits = o.matmul_ordered(codes.astype(np.float32) * scales[:, None], self.w)
        sel, wts = o.select_top_k(logits, self.k)
        return (torch.from_numpy(codes), torch.from_numpy(scales), torch.from_numpy(sel.astype(np.int64)),
                torch.from_numpy(wts.astype(np.float32)))

    def experts(self, codes, scales, eid, n_local):
        codes, scales, eid = codes.numpy(), scales.numpy(), eid.numpy()
        d = self.local[0][2][0].shape[0]
        out = np.zeros((codes.shape[0], d), np.float32)
        for e in range(n_local):
            rows = np.nonzero(eid == e)[0]
            if rows.size == 0:
                continue
            (cg, ig, gg), (cu, iu, gu), (cd, idn, gd) = self.local[e]
            a = o.lut_gemm(codes[rows], scales[rows], ig, cg, gg)
            b = o.lut_gemm(codes[rows], scales[rows], iu, cu, gu)
            hc, hs = o.quantize((o.silu(a) * b).astype(np.float32), 4)
            out[rows] = o.lut_gemm(hc, hs, idn, cd, gd)
        return torch.from_numpy(out)

    def combine(self, selected, weights, f_routes):
        sel, w, f = selected.numpy(), weights.numpy(), f_routes.numpy()
        n, k = sel.shape
        out = np.zeros((n, f.shape[1]), np.float32)
        for t in range(n):
            for s in np.argsort(sel[t], kind="stable"):
                out[t] = out[t] + w[t, s] * f[t * k + s]
        return torch.from_numpy(out)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seed, n, d, ff, E, k, g = cfg
        v, w, experts, _ = moe_inputs_host(seed, n, d, ff, E, g)
        begin, per = expert_range(E, world, rank)
        be = OracleBackend(w, experts[begin:begin + per])
        be.k = k
        layer = EPMoE(be, E, k, rank, world)
        lo, hi = rank * n // world, (rank + 1) * n // world
        out = layer(torch.from_numpy(v[lo:hi]))
        result_q.put((rank, out.numpy()))
    except Exception as exc:  # surface the failure instead of a queue timeout
        result_q.put((rank, repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [(3, 24, 64, 96, 4, 2, 32), (7, 17, 128, 64, 6, 3, 64)])
def test_ep_world2_matches_single_process_oracle(cfg):
    seed, n, d, ff, E, k, g = cfg
    if E % 2:
        pytest.skip("experts must split evenly")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = dict(q.get(timeout=120) for _ in range(2))
    for r in range(2):
        assert not isinstance(parts[r], str), parts[r]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([parts[0], parts[1]])
    v, w, experts, _ = moe_inputs_host(seed, n, d, ff, E, g)
    want = o.moe_layer(v, w, experts, k)
    assert np.array_equal(got.view(np.int32), want.view(np.int32))


def test_plan_dispatch_orders_routes_by_destination():
    sel = torch.tensor([[3, 0], [1, 2], [0, 3], [2, 1]])
    order, dest, counts = plan_dispatch(sel, n_experts=4, world=2)
    assert counts.tolist() == [4, 4]
    assert dest.tolist() == [0] * 4 + [1] * 4
    # stable: routes to each rank keep (token, slot) order
    flat = sel.reshape(-1)
    assert flat[order].tolist() == [0, 1, 0, 1, 3, 2, 3, 2]
