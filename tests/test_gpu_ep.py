"""The expert-parallel driver on the CUDA backend (NCCL, world_size 1 on the
single GPU this run has; the multi-rank exchange logic is covered by the gloo
tests).  Routing, segment order and per-row arithmetic are the same as the
single-GPU layer, so the outputs must be bitwise equal."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu

from paper_2604_10496_b200.ep import CudaBackend, EPMoE, EPStep  # noqa: E402
from paper_2604_10496_b200.moe import ExpertStack, MoELayer  # noqa: E402
from paper_2604_10496_b200.synthetic import moe_inputs_device  # noqa: E402


@pytest.fixture(scope="module")
def nccl_world1():
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("path", ["tc", "f32"])
def test_ep_world1_equals_single_gpu_layer(nccl_world1, path):
    n, d, ff, E, k, g = 48, 1024, 1536, 8, 2, 128
    v, w, sites, _ = moe_inputs_device(5, n, d, ff, E, g)
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, path=path)
    if path == "tc":
        layer.prepare_tc()
    want = layer(v).clone()
    ep = EPMoE(CudaBackend(layer), E, k, rank=0, world=1)
    got = ep(v)
    torch.cuda.synchronize()
    assert torch.equal(got, want)


def _shard(stack, begin, per):
    return ExpertStack(stack.ids[begin:begin + per].contiguous(), stack.centroids[begin:begin + per].contiguous(),
                       stack.d_in, stack.d_out, stack.group_size)


@pytest.mark.parametrize("world,n_tok,E,k", [(2, 40, 8, 2), (4, 33, 8, 2), (2, 21, 6, 3)])
def test_ep_sharded_ranks_in_one_process(world, n_tok, E, k):
    """`world` ranks with E/world experts each, driven in one process: the
    all_to_all exchanges are done here by concatenating the send segments.
    Each rank's layer holds only its experts (expert_begin/n_local < E), so
    this runs the sharded route/expert/combine kernels exactly as a real
    multi-GPU run would."""
    d, ff, g = 1024, 1536, 128
    v, w, sites, _ = moe_inputs_device(11, n_tok, d, ff, E, g)
    full = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    ref = MoELayer.from_stacks(w, *full, top_k=k, path="tc")
    ref.prepare_tc()
    want = ref(v).clone()
    per = E // world
    ranks = []
    for r in range(world):
        loc = MoELayer.from_stacks(w, *(_shard(s, r * per, per) for s in full), top_k=k, path="tc",
                                   expert_begin=r * per, n_experts=E)
        loc.prepare_tc()
        ranks.append(EPMoE(CudaBackend(loc), E, k, rank=r, world=world))
    bounds = [(r * n_tok // world, (r + 1) * n_tok // world) for r in range(world)]
    states = [ep.dispatch(v[lo:hi]) for ep, (lo, hi) in zip(ranks, bounds)]
    cuts = [np.concatenate([[0], np.cumsum(st["send"].tolist())]) for st in states]

    def seg(st, c, key, q):
        return st[key][int(c[q]):int(c[q + 1])]

    back = [[None] * world for _ in range(world)]
    for q, ep in enumerate(ranks):
        parts = {key: torch.cat([seg(st, c, key, q) for st, c in zip(states, cuts)]) for key in ("codes", "scales",
                                                                                                 "eid")}
        f = ep.compute(parts["codes"], parts["scales"], parts["eid"])
        off = 0
        for r, (st, c) in enumerate(zip(states, cuts)):
            cnt = int(c[q + 1] - c[q])
            back[r][q] = f[off:off + cnt]
            off += cnt
    got = torch.cat([ep.finish(st, torch.cat(back[r])) for r, (ep, st) in enumerate(zip(ranks, states))])
    torch.cuda.synchronize()
    assert torch.equal(got, want)


def _sharded_layers(w, full, E, k, world, path="tc"):
    per = E // world
    out = []
    for r in range(world):
        loc = MoELayer.from_stacks(w, *(_shard(s, r * per, per) for s in full), top_k=k, path=path,
                                   expert_begin=r * per, n_experts=E)
        if path == "tc":
            loc.prepare_tc()
        out.append(loc)
    return out


def _run_ranks_in_process(steps, xs):
    """Drive EPStep phases of all ranks, doing the two equal-split exchanges
    by slicing: recv_q[src block] = send_src[q block]."""
    world, cap = len(steps), steps[0].cap
    for st, x in zip(steps, xs):
        st.route_and_pack(x)
    for q, st in enumerate(steps):
        for src, other in enumerate(steps):
            st.recv[src * cap:(src + 1) * cap].copy_(other.send[q * cap:(q + 1) * cap])
    for st in steps:
        st.run_experts()
    for r, st in enumerate(steps):
        for q, other in enumerate(steps):
            st.ret[q * cap:(q + 1) * cap].copy_(other.back[r * cap:(r + 1) * cap])
    return [st.combine().clone() for st in steps]


@pytest.mark.parametrize("world,n_tok,E,k,path", [(2, 40, 8, 2, "tc"), (4, 32, 8, 2, "tc"), (8, 16, 8, 2, "tc"),
                                                  (2, 21, 6, 3, "tc"), (2, 24, 8, 2, "f32")])
def test_ep_step_slots_match_single_gpu_layer(world, n_tok, E, k, path):
    """Fixed-capacity EP step (device-side dispatch / group / scatter): every
    rank's combined output equals the single-GPU layer's rows bit for bit."""
    d, ff, g = 1024, 1536, 128
    v, w, sites, _ = moe_inputs_device(13, n_tok * world, d, ff, E, g)
    full = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    ref = MoELayer.from_stacks(w, *full, top_k=k, path=path)
    if path == "tc":
        ref.prepare_tc()
    want = ref(v).clone()
    layers = _sharded_layers(w, full, E, k, world, path)
    steps = [EPStep(layers[r], n_tok, r, world, all_to_all=lambda o, i: None) for r in range(world)]
    got = torch.cat(_run_ranks_in_process(steps, [v[r * n_tok:(r + 1) * n_tok] for r in range(world)]))
    torch.cuda.synchronize()
    assert torch.equal(got, want)


def test_ep_step_unpacked_slots_for_odd_width():
    """d_model % 32 != 0 (1040) sends int8 codes instead of packed nibbles; the
    step is still bitwise equal to the single-GPU layer (fp32 path, g = 16)."""
    world, n_tok, E, k, d, ff, g = 2, 20, 8, 2, 1040, 256, 16
    v, w, sites, _ = moe_inputs_device(37, n_tok * world, d, ff, E, g)
    full = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    ref = MoELayer.from_stacks(w, *full, top_k=k, path="f32")
    want = ref(v).clone()
    layers = _sharded_layers(w, full, E, k, world, "f32")
    steps = [EPStep(layers[r], n_tok, r, world, all_to_all=lambda o, i: None) for r in range(world)]
    assert steps[0].send.shape[-1] == d + 16  # int8 codes
    got = torch.cat(_run_ranks_in_process(steps, [v[r * n_tok:(r + 1) * n_tok] for r in range(world)]))
    torch.cuda.synchronize()
    assert torch.equal(got, want)


@pytest.mark.parametrize("geometry", ["prefill", "decode"])
@pytest.mark.parametrize("world,n_tok", [(4, 48), (8, 32)])
def test_ep_step_rank_gemm_geometries(monkeypatch, geometry, world, n_tok):
    """The per-rank expert GEMMs with the slot capacity as the row bound and the
    routed row count on the device, in either geometry (4 and 8 GPUs take the
    prefill geometry at Mixtral size): bitwise equal to the single-GPU layer."""
    E, k, d, ff, g = 8, 2, 1024, 1536, 128
    v, w, sites, _ = moe_inputs_device(29 + world, n_tok * world, d, ff, E, g)
    full = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    ref = MoELayer.from_stacks(w, *full, top_k=k, path="tc")
    ref.prepare_tc()
    want = ref(v).clone()
    monkeypatch.setenv("CQ_UMMA_GEOMETRY", geometry)
    layers = _sharded_layers(w, full, E, k, world)
    steps = [EPStep(layers[r], n_tok, r, world, all_to_all=lambda o, i: None) for r in range(world)]
    assert steps[0].send.shape[-1] == d // 2 + 16  # codes as packed nibbles
    got = torch.cat(_run_ranks_in_process(steps, [v[r * n_tok:(r + 1) * n_tok] for r in range(world)]))
    torch.cuda.synchronize()
    assert torch.equal(got, want)


def test_ep_step_skewed_routing_fills_one_rank():
    """All tokens routed to the experts of rank 0 (router columns of the other
    ranks pushed to -inf-like values): rank 0's slots fill to capacity, the
    other ranks receive nothing and run no expert rows."""
    world, n_tok, E, k, d, ff, g = 4, 16, 8, 2, 1024, 1536, 128
    v, w, sites, _ = moe_inputs_device(17, n_tok * world, d, ff, E, g)
    w = w.clone()
    w[:, 2:] = -1e3 * w[:, 2:].abs() - 1.0   # experts 0, 1 (rank 0) always win
    v = v.abs() + 0.01                        # positive inputs keep the margin
    full = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    ref = MoELayer.from_stacks(w, *full, top_k=k, path="tc")
    ref.prepare_tc()
    want = ref(v).clone()
    assert set(ref.trace(n_tok * world)["selected"].unique().tolist()) <= {0, 1}
    layers = _sharded_layers(w, full, E, k, world)
    steps = [EPStep(layers[r], n_tok, r, world, all_to_all=lambda o, i: None) for r in range(world)]
    got = torch.cat(_run_ranks_in_process(steps, [v[r * n_tok:(r + 1) * n_tok] for r in range(world)]))
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    assert steps[0].offsets[-1].item() == n_tok * world * k
    assert all(st.offsets[-1].item() == 0 for st in steps[1:])


def test_ep_step_world1_nccl_graph_capture(nccl_world1):
    """The whole EP step (NCCL all_to_all included) captured in a CUDA graph
    and replayed equals the eager single-GPU layer."""
    n, d, ff, E, k, g = 32, 1024, 1536, 8, 2, 128
    v, w, sites, _ = moe_inputs_device(23, n, d, ff, E, g)
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, path="tc")
    layer.prepare_tc()
    want = layer(v).clone()
    step = EPStep(layer, n, 0, 1)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        eager = step(v).clone()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            step(v)
        step.out.zero_()
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(eager, want)
    assert torch.equal(step.out, want)


@pytest.mark.parametrize("i", range(6))
def test_ep_step_random_shapes(i):
    """Random world size, expert count, top-k, batch and width: the sharded EP
    step (in-process ranks) bitwise equal to the single-GPU layer."""
    rng = np.random.default_rng(700 + i)
    world = int(rng.choice([2, 4, 8]))
    E = world * int(rng.choice([1, 2, 4]))
    k = int(rng.integers(1, min(4, E) + 1))
    n_tok = int(rng.choice([1, 7, 32, 50]))
    d = int(rng.choice([512, 1024]))
    ff, g = 512, 128
    v, w, sites, _ = moe_inputs_device(800 + i, n_tok * world, d, ff, E, g)
    full = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    ref = MoELayer.from_stacks(w, *full, top_k=k, path="tc")
    ref.prepare_tc()
    want = ref(v).clone()
    layers = _sharded_layers(w, full, E, k, world)
    steps = [EPStep(layers[r], n_tok, r, world, all_to_all=lambda o, i: None) for r in range(world)]
    got = torch.cat(_run_ranks_in_process(steps, [v[r * n_tok:(r + 1) * n_tok] for r in range(world)]))
    torch.cuda.synchronize()
    assert torch.equal(got, want)
