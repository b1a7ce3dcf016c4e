"""The expert-parallel step on the B200 kernels (ep.EPStep, csrc/ep.cu).

This run has one GPU, so multi-rank steps are driven here as in-process
ranks: every rank's phases run on the real kernels with its own sharded
layer (expert_begin / n_local < E), and the two exchanges are done by slicing
the send buffers exactly as all_to_all(-v) would.  A true 2-process run on the
one GPU (exchanges staged through host memory over gloo) and an NCCL world-1
run cover the step's own stream/exchange orchestration.

Parity: the exact-row protocol is bitwise equal to the single-GPU layer; the
dedup protocol equals it up to fp32 re-association of the cross-rank adds
(bitwise for tokens whose experts share a rank); the device send rows equal
ep.pack_rows (the protocol restated in torch, checked against the oracle on
CPU by tests/test_ep_gloo.py) byte for byte."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

from paper_2604_10496_b200.ep import EPStep, pack_rows, plan_rows  # noqa: E402
from paper_2604_10496_b200.moe import ExpertStack, MoELayer  # noqa: E402
from paper_2604_10496_b200.synthetic import moe_inputs_device  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def nccl_world1():
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def _stacks(sites, g):
    return [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]


def _shard(stack, begin, per):
    return ExpertStack(stack.ids[begin:begin + per].contiguous(), stack.centroids[begin:begin + per].contiguous(),
                       stack.d_in, stack.d_out, stack.group_size)


def _build(seed, n_all, d, ff, E, k, g, n_sh=0, path="tc"):
    v, w, sites, sh = moe_inputs_device(seed, n_all, d, ff, E, g, n_shared=n_sh)
    full = _stacks(sites, g)
    shared = tuple(_stacks(sh, g)) if n_sh else None
    ref = MoELayer.from_stacks(w, *full, top_k=k, shared=shared, path=path)
    if path == "tc":
        ref.prepare_tc()
    return v, w, full, shared, ref


def _sharded_layers(w, full, shared, E, k, world, path="tc"):
    per = E // world
    out = []
    for r in range(world):
        loc = MoELayer.from_stacks(w, *(_shard(s, r * per, per) for s in full), top_k=k, shared=shared, path=path,
                                   expert_begin=r * per, n_experts=E)
        if path == "tc":
            loc.prepare_tc()
        out.append(loc)
    return out


def _sim_a2a(outs, ins, splits, cap):
    """outs[q] = concat over sources src of ins[src]'s block for q (all_to_all(-v))."""
    world = len(ins)
    for q in range(world):
        parts = []
        for src in range(world):
            sp = splits[src] if splits[src] is not None else [cap] * world
            lo = sum(sp[:q])
            parts.append(ins[src][lo:lo + sp[q]])
        cat = torch.cat(parts)
        outs[q][:cat.shape[0]].copy_(cat)


def _run_in_process(steps, xs):
    world = len(steps)
    for st, x in zip(steps, xs):
        st.dispatch(x)
    if steps[0].sizing == "compact":
        for q, st in enumerate(steps):
            for src, other in enumerate(steps):
                st.rcounts[src].copy_(other.counts[q])
        for st in steps:
            st.read_counts()
    for st in steps:
        st.run_shared()
    cap = steps[0].cap
    for m in range(steps[0].M):
        views = [st.views(m) for st in steps]
        _sim_a2a([v[1] for v in views], [v[0] for v in views], [st.splits(m)[0] for st in steps], cap)
        for st in steps:
            st.experts(m)
        _sim_a2a([v[3] for v in views], [v[2] for v in views], [st.splits(m)[1] for st in steps], cap)
    outs = []
    for st in steps:
        for m in range(st.M):
            st.combine(m, st.out)
        outs.append(st.out.clone())
    assert world == len(outs)
    return torch.cat(outs)


def _check(got, want, dedup, ref=None, n_all=None, E=None, world=None):
    if not dedup:
        assert torch.equal(got, want)
        return
    g64, w64 = got.double(), want.double()
    rel = float((g64 - w64).norm() / w64.norm())
    assert rel <= 1e-6, rel
    if ref is not None:  # tokens whose experts all live on one rank: bitwise
        sel = ref.trace(n_all)["selected"]
        one = (sel // (E // world) == (sel[:, :1] // (E // world))).all(1)
        assert torch.equal(got[one], want[one])


CASES = {  # name: (n per rank, d, ff, E, k, n_shared, world)
    "mx_w2": (24, 1024, 1536, 8, 2, 0, 2),
    "mx_w8": (16, 1024, 1536, 8, 2, 0, 8),
    "qw_w2": (24, 2048, 768, 128, 8, 0, 2),
    "qw_w4": (20, 2048, 768, 128, 8, 0, 4),
    "qw_w8": (16, 2048, 768, 128, 8, 0, 8),
    "ds_w8": (24, 2048, 1408, 64, 6, 2, 8),
    "ds_w2": (20, 2048, 1408, 64, 6, 2, 2),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("dedup,sizing,mb", [(False, "fixed", 1), (True, "compact", 2), (True, "fixed", 1)])
def test_ep_step_matches_single_gpu_layer(case, dedup, sizing, mb):
    """QW (128 experts, top-8) and DS (64 + 2 shared, top-6) at world 2/4/8,
    Mixtral-shaped at 2/8: every rank's output against the single-GPU layer."""
    n, d, ff, E, k, n_sh, world = CASES[case]
    g = 128
    v, w, full, shared, ref = _build(41 + world, n * world, d, ff, E, k, g, n_sh)
    want = ref(v).clone()
    layers = _sharded_layers(w, full, shared, E, k, world)
    steps = [EPStep(layers[r], n, r, world, dedup=dedup, sizing=sizing, micro_batches=mb, exchange=lambda *a: None)
             for r in range(world)]
    got = _run_in_process(steps, [v[r * n:(r + 1) * n] for r in range(world)])
    torch.cuda.synchronize()
    _check(got, want, dedup, ref, n * world, E, world)


@pytest.mark.parametrize("dedup", [True, False])
def test_ep_send_rows_equal_protocol_bytes(dedup):
    """Compact sizing: the device rows (codes as nibbles, scale, routes,
    weights) equal ep.pack_rows(plan_rows(...)) byte for byte; counts and
    src_slot / src_w equal the plan's."""
    n, d, ff, E, k, world, g = 40, 2048, 768, 64, 6, 4, 128
    v, w, full, _, _ = _build(61, n * world, d, ff, E, k, g)
    layers = _sharded_layers(w, full, None, E, k, world)
    for r in (0, 3):
        st = EPStep(layers[r], n, r, world, dedup=dedup, sizing="compact", exchange=lambda *a: None)
        st.dispatch(v[r * n:(r + 1) * n])
        tr = st.tr
        p = plan_rows(tr["selected"], tr["weights"], E, world, dedup)
        want = pack_rows(tr["codes"], tr["scales"], p)
        assert torch.equal(st.send[0][:want.shape[0]], want)
        assert torch.equal(st.counts[:, 0, 0], p.counts) and torch.equal(st.counts[:, 0, 1], p.routes)
        assert torch.equal(st.src_slot[0], p.src_slot) and torch.equal(st.src_w[0], p.src_w)


def test_ep_dedup_moves_fewer_bytes_than_exact():
    """DS at world 8: one row per (token, peer) — the exchange shrinks from one
    row per route (top-6) to ~4.5 rows per token, both directions."""
    n, d, ff, E, k, n_sh, world = CASES["ds_w8"]
    v, w, full, shared, _ = _build(43, n * world, d, ff, E, k, 128, n_sh)
    layers = _sharded_layers(w, full, shared, E, k, world)
    res = {}
    for dedup in (True, False):
        steps = [EPStep(layers[r], n, r, world, dedup=dedup, sizing="compact", exchange=lambda *a: None)
                 for r in range(world)]
        _run_in_process(steps, [v[r * n:(r + 1) * n] for r in range(world)])
        res[dedup] = sum(st.exchange_bytes()["back"] for st in steps)
    assert res[True] < 0.85 * res[False]


def test_ep_step_unpacked_rows_for_odd_width():
    """d_model % 32 != 0 (1040) sends int8 codes instead of packed nibbles; still
    bitwise equal to the single-GPU layer (fp32 path, g = 16, exact rows)."""
    world, n, E, k, d, ff, g = 2, 20, 8, 2, 1040, 256, 16
    v, w, full, _, ref = _build(37, n * world, d, ff, E, k, g, path="f32")
    want = ref(v).clone()
    layers = _sharded_layers(w, full, None, E, k, world, "f32")
    steps = [EPStep(layers[r], n, r, world, dedup=False, exchange=lambda *a: None) for r in range(world)]
    assert steps[0].rb == d + 16
    got = _run_in_process(steps, [v[r * n:(r + 1) * n] for r in range(world)])
    torch.cuda.synchronize()
    assert torch.equal(got, want)


@pytest.mark.parametrize("geometry", ["prefill", "decode"])
def test_ep_step_rank_gemm_geometries(monkeypatch, geometry):
    """The per-rank expert GEMMs in either geometry: bitwise equal to the single-GPU layer."""
    world, n, E, k, d, ff, g = 4, 48, 8, 2, 1024, 1536, 128
    v, w, full, _, ref = _build(33, n * world, d, ff, E, k, g)
    want = ref(v).clone()
    monkeypatch.setenv("CQ_UMMA_GEOMETRY", geometry)
    layers = _sharded_layers(w, full, None, E, k, world)
    steps = [EPStep(layers[r], n, r, world, dedup=False, exchange=lambda *a: None) for r in range(world)]
    got = _run_in_process(steps, [v[r * n:(r + 1) * n] for r in range(world)])
    torch.cuda.synchronize()
    assert torch.equal(got, want)


@pytest.mark.parametrize("sizing", ["fixed", "compact"])
def test_ep_step_skewed_routing_fills_one_rank(sizing):
    """All tokens routed to rank 0's experts: its slots fill to capacity, the
    other ranks receive nothing and run no expert rows."""
    world, n, E, k, d, ff, g = 4, 16, 8, 2, 1024, 1536, 128
    v, w, sites, _ = moe_inputs_device(17, n * world, d, ff, E, g)
    w = w.clone()
    w[:, 2:] = -1e3 * w[:, 2:].abs() - 1.0   # experts 0, 1 (rank 0) always win
    v = v.abs() + 0.01                        # positive inputs keep the margin
    full = _stacks(sites, g)
    ref = MoELayer.from_stacks(w, *full, top_k=k, path="tc").prepare_tc()
    want = ref(v).clone()
    assert set(ref.trace(n * world)["selected"].unique().tolist()) <= {0, 1}
    layers = _sharded_layers(w, full, None, E, k, world)
    steps = [EPStep(layers[r], n, r, world, dedup=True, sizing=sizing, exchange=lambda *a: None)
             for r in range(world)]
    got = _run_in_process(steps, [v[r * n:(r + 1) * n] for r in range(world)])
    torch.cuda.synchronize()
    assert torch.equal(got, want)   # one destination rank per token: dedup is bitwise here
    assert steps[0].offsets[-1].item() == n * world * k
    assert all(st.offsets[-1].item() == 0 for st in steps[1:])


@pytest.mark.parametrize("dedup,sizing,mb", [(False, "fixed", 1), (True, "fixed", 2), (True, "compact", 3)])
def test_ep_step_world1_nccl(nccl_world1, dedup, sizing, mb):
    """The whole step through NCCL (world 1, DS-shaped with shared experts,
    micro-batches on the communication stream): bitwise equal to the layer;
    fixed sizing also captured in a CUDA graph and replayed."""
    n, d, ff, E, k, g, n_sh = 48, 1024, 1024, 8, 3, 128, 2
    v, w, full, shared, ref = _build(23, n, d, ff, E, k, g, n_sh)
    want = ref(v).clone()
    step = EPStep(ref, n, 0, 1, dedup=dedup, sizing=sizing, micro_batches=mb)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        eager = step(v).clone()
        if sizing == "fixed":
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=s):
                step(v)
            step.out.zero_()
            graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(eager, want)
    if sizing == "fixed":
        assert torch.equal(step.out, want)


def _gloo_rank(rank, world, port, q):
    """One rank of a 2-process EP step on the single GPU: exchanges staged
    through host memory over gloo (the kernels of the two ranks never wait on
    each other; only the host exchange joins them)."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        n, d, ff, E, k, g, n_sh = 32, 2048, 1408, 64, 6, 128, 2
        v, w, full, shared, ref = _build(71, n * world, d, ff, E, k, g, n_sh)
        want = ref(v).clone()
        layers = _sharded_layers(w, full, shared, E, k, world)

        def host_a2a(out, inp, out_splits, in_splits):
            torch.cuda.current_stream().synchronize()
            h_out = torch.empty(out.shape, dtype=out.dtype)
            dist.all_to_all_single(h_out, inp.cpu(), out_splits, in_splits)
            out.copy_(h_out)

        res = {}
        for dedup, sizing, mb in ((False, "fixed", 1), (True, "compact", 2)):
            step = EPStep(layers[rank], n, rank, world, dedup=dedup, sizing=sizing, micro_batches=mb,
                          exchange=host_a2a)
            got = step(v[rank * n:(rank + 1) * n]).clone()
            torch.cuda.synchronize()
            mine = want[rank * n:(rank + 1) * n]
            rel = float((got.double() - mine.double()).norm() / mine.double().norm())
            res[(dedup, sizing)] = (bool(torch.equal(got, mine)), rel)
        q.put((rank, res))
    except Exception as exc:
        q.put((rank, repr(exc)))
        raise
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_ep_step_two_processes_gloo_staged():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
    for r in range(2):
        assert not isinstance(res[r], str), res[r]
        assert res[r][(False, "fixed")][0], res[r]          # exact rows: bitwise
        assert res[r][(True, "compact")][1] <= 1e-6, res[r]  # dedup: fp32 re-association


@pytest.mark.parametrize("i", range(6))
def test_ep_step_random_shapes(i):
    """Random world size, expert count, top-k, batch, width, shared experts,
    protocol and sizing: the in-process EP step against the single-GPU layer."""
    rng = np.random.default_rng(700 + i)
    world = int(rng.choice([2, 4, 8]))
    E = world * int(rng.choice([1, 2, 4]))
    k = int(rng.integers(1, min(6, E) + 1))
    n = int(rng.choice([1, 7, 32, 50]))
    d = int(rng.choice([512, 1024]))
    n_sh = int(rng.integers(0, 3))
    dedup, sizing, mb = bool(rng.integers(0, 2)), str(rng.choice(["fixed", "compact"])), int(rng.integers(1, 4))
    v, w, full, shared, ref = _build(800 + i, n * world, d, 512, E, k, 128, n_sh)
    want = ref(v).clone()
    layers = _sharded_layers(w, full, shared, E, k, world)
    steps = [EPStep(layers[r], n, r, world, dedup=dedup, sizing=sizing, micro_batches=mb, exchange=lambda *a: None)
             for r in range(world)]
    got = _run_in_process(steps, [v[r * n:(r + 1) * n] for r in range(world)])
    torch.cuda.synchronize()
    _check(got, want, dedup, ref, n * world, E, world)
