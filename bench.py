#!/usr/bin/env python
"""Benchmark: MoE-layer tokens/s of the CodeQuant Stage-4 LUT MoE path on B200.

Workload (BASELINE.json configs[1]): Mixtral-8x7B MoE layer shape — d_model
4096, d_ff 14336, 8 experts, top-2, 16-centroid codebooks with group size 128,
decode batch 64 tokens, random-init codebook weights (1.41 GB, larger than the
126 MB L2, so no flush is needed between steps).  One step = one MoE-layer
forward over one batch: quantize -> ordered router -> top-k -> permute ->
grouped gate|up LUT GEMM + silu -> re-quantize -> grouped down -> combine.

    python bench.py [--gpus N --steps K --warmup W --batch B --path auto|tc|f32]
    python bench.py --impl reference ...   # the reference CPU kernel (oracle/_ref)

N > 1 (torchrun): expert parallelism (ep.py; `run_ep`): E/N experts and a
batch of B tokens per rank, NCCL all_to_all dispatch/return, reported as weak
scaling; time = max over ranks.  `--replicas` runs N independent full layers
instead; `--ep` forces the EP driver at N = 1 (torchrun --nproc-per-node 1).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# SURVEY.md §8(d) configurations.  The headline (default) is MX: the Mixtral-8x7B
# layer at decode batch 64 (BASELINE.json configs[1]); the others are for the
# per-config table in DESIGN.md and are selected with --config.
CONFIGS = {
    "mx": dict(name="mixtral-8x7b-moe-layer-decode", d_model=4096, d_ff=14336, n_experts=8, top_k=2, batch=64),
    "mx1": dict(name="mixtral-8x7b-moe-layer-decode-b1", d_model=4096, d_ff=14336, n_experts=8, top_k=2, batch=1),
    "mx8": dict(name="mixtral-8x7b-moe-layer-decode-b8", d_model=4096, d_ff=14336, n_experts=8, top_k=2, batch=8),
    "mxe": dict(name="mixtral-8x7b-moe-layer-decode-embedding-wise", d_model=4096, d_ff=14336, n_experts=8,
                top_k=2, batch=64, group_size=0),
    "mx3": dict(name="mixtral-8x7b-moe-layer-decode-w3", d_model=4096, d_ff=14336, n_experts=8, top_k=2,
                batch=64, kc=8),
    "mx2": dict(name="mixtral-8x7b-moe-layer-decode-w2", d_model=4096, d_ff=14336, n_experts=8, top_k=2,
                batch=64, kc=4),
    "c1": dict(name="c1-moe-layer-cpu-parity", d_model=1024, d_ff=2816, n_experts=8, top_k=2, batch=64),
    "ph": dict(name="phi-3.5-moe-layer-prefill-rotation", d_model=4096, d_ff=6400, n_experts=16, top_k=2,
               batch=4096, rotation=True),
    "qw": dict(name="qwen3-30b-a3b-moe-layer-prefill", d_model=2048, d_ff=768, n_experts=128, top_k=8, batch=4096),
    "qw64": dict(name="qwen3-30b-a3b-moe-layer-decode", d_model=2048, d_ff=768, n_experts=128, top_k=8, batch=64),
    # SURVEY 8(d)'s QW sizes for the scaling rows: decode N = 256, strong-scaling prefill N = 8192
    "qw256": dict(name="qwen3-30b-a3b-moe-layer-decode-256", d_model=2048, d_ff=768, n_experts=128, top_k=8,
                  batch=256),
    "qw8k": dict(name="qwen3-30b-a3b-moe-layer-prefill-8192", d_model=2048, d_ff=768, n_experts=128, top_k=8,
                 batch=8192),
    "ds": dict(name="deepseek-v2-lite-moe-block-prefill", d_model=2048, d_ff=1408, n_experts=64, top_k=6,
               batch=8192, n_shared=2),
}
CFG = dict(CONFIGS["mx"], group_size=128)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="mx", choices=sorted(CONFIGS))
    p.add_argument("--batch", type=int, default=None, help="tokens per step (per rank); default: the config's")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--path", default="auto", choices=["auto", "tc", "f32", "ordered"])
    p.add_argument("--layout", default="umma128u", choices=["umma128u"],
                   help="tensor-core weight layout / kernel")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--replicas", action="store_true",
                   help="N > 1: independent full replicas instead of expert parallelism")
    p.add_argument("--ep", action="store_true", help="expert-parallel driver even at N = 1 (under torchrun)")
    p.add_argument("--seed", type=int, default=0)
    return p.parse_args()


def layer_bytes(n_active: int, R: int) -> dict:
    """Algorithmic HBM bytes for R routed rows: reference-format
    weights of the active experts + activations, per layer and for the gate|up
    kernel."""
    d, ff, g = CFG["d_model"], CFG["d_ff"], CFG["group_size"]
    w_gu = 2 * (ff * d // 2 + ff * (d // (g or d)) * 16 * 4)  # gate + up ids + centroids (g = 0: g = d_in)
    w_dn = d * ff // 2 + d * (ff // (g or ff)) * 16 * 4
    gu = n_active * w_gu + R * d + R * 4 + R * ff * 4         # + codes, scales in; hidden out
    dn = n_active * w_dn + R * ff + R * 4 + R * d * 4
    return dict(gate_up=gu, down=dn, layer=gu + dn + d * CFG["n_experts"] * 4)


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled during the timed region.

    NVML polled from a thread every ~2 ms (nvidia-smi's 100 ms loop is too slow
    for a millisecond-scale region); falls back to nvidia-smi if NVML is absent.
    """

    def __init__(self, index: int):
        self.index, self.rows, self.stop, self.thread = index, [], threading.Event(), None
        self.ready = threading.Event()

    def _poll_nvml(self):
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        names = {nv.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                 nv.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                 nv.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                 nv.nvmlClocksEventReasonSwPowerCap: "sw_power_cap",
                 nv.nvmlClocksEventReasonHwPowerBrakeSlowdown: "hw_power_brake"}
        while not self.stop.is_set():
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.rows.append((sm, mx, [v for k, v in names.items() if bits & k]))
            self.ready.set()
            time.sleep(0.002)
        nv.nvmlShutdown()

    def __enter__(self):
        try:
            import pynvml  # noqa: F401
            self.thread = threading.Thread(target=self._poll_nvml, daemon=True)
            self.thread.start()
            self.ready.wait(timeout=5.0)   # NVML init can take longer than a short timed region
            self.rows.clear()
        except ImportError:
            self.thread = None
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [r[0] for r in self.rows]
        reasons = sorted({x for r in self.rows for x in r[2]})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(self.rows[0][1]),
                "reasons": reasons, "samples": len(self.rows), "source": "nvml"}


SPEC_HBM_GBS, SPEC_BF16_TFLOPS = 8000.0, 2250.0  # B200 data-sheet HBM3e bandwidth, dense bf16


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        # burst bf16 peak: every kernel here is event-timed alone, well under the sustained-power regime
        return {"hbm_gbs": p["hbm_gbs"], "bf16_tflops": p["bf16_tflops"],
                "bf16_tflops_sustained": p.get("bf16_tflops_sustained"), "src": "measured"}
    except (OSError, KeyError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 2250.0, "src": "fallback"}


# ---------------------------------------------------------------------------
# CPU side: the reference's own kernel (oracle/_ref) on the host cores.


def host_layer(seed: int, n: int):
    rng = np.random.default_rng(seed)
    d, ff, E, g = CFG["d_model"], CFG["d_ff"], CFG["n_experts"], CFG["group_size"]
    v = rng.standard_normal((n, d)).astype(np.float32)
    w = (rng.standard_normal((d, E)) / math.sqrt(d)).astype(np.float32)
    experts = []
    for _ in range(E):
        mats = []
        for di, do in ((d, ff), (d, ff), (ff, d)):
            gs = g or di
            mats.append(((rng.standard_normal((do, di // gs, 16), dtype=np.float32) / math.sqrt(di)),
                         rng.integers(0, 256, (do, di // 2), dtype=np.uint8), gs))
        experts.append(mats)
    return v, w, experts


def _row_slices(rows: int, parts: int):
    step = -(-rows // parts)
    return [(r0, min(r0 + step, rows)) for r0 in range(0, rows, step)]


_REF_EXPERTS = None  # the host layer's experts, inherited by the forked workers (copy-on-write)


def _ref_gemm_task(e, site, r0, r1, q, s):
    """Worker: the reference's _core.lut_gemm_f32 on output rows [r0, r1) of
    expert e's `site` matrix, all of the expert's tokens in one block."""
    import oracle
    cent, ids, g = _REF_EXPERTS[e][site]
    out = np.zeros((q.shape[0], r1 - r0), np.float32)
    oracle.ref_core().lut_gemm_f32(q, s, ids[r0:r1], cent[r0:r1], g, max(q.shape[0], 1), out, 0, q.shape[0])
    return out


def cpu_reference_layer(v, w, experts, k, pool, parts):
    """One FULL composed MoE block (model.py:377-404) on the
    reference's native kernels (oracle/_ref, built from its _core.pyx):
    quantize_activations (quant.py:89-100) -> _core.matmul_f32 router ->
    select_top_k -> per active expert _core.lut_gemm_f32 for gate and up ->
    silu * up -> quantize -> _core.lut_gemm_f32 for down -> weighted sum in
    ascending expert order.  All experts, all rows, every token.

    Parallelism: the reference threads a GEMM over token blocks
    (kernels/compiled.py:27-51), which at decode (~16 tokens per expert) only
    re-builds every row's tables per block; here its kernel runs on disjoint
    OUTPUT-ROW slices of each expert matrix instead (all of the expert's tokens
    in one block, one writer per output element, so bitwise the same result),
    every GEMM of a stage in flight at once, on a pool of one forked worker
    process per host core (the kernel's nogil threads did not scale on every
    host we measured; processes do).  `experts` must be the module-level
    _REF_EXPERTS the pool was forked with."""
    import oracle
    from oracle import oracle as o
    core = oracle.ref_core()
    n = v.shape[0]
    codes, scales = o.quantize(v, 4)
    logits = np.zeros((n, w.shape[1]), np.float32)
    core.matmul_f32(np.ascontiguousarray(codes.astype(np.float32) * scales[:, None]), w, logits)
    sel, wts = o.select_top_k(logits, k)

    def gemm_jobs(e, site, q, s):
        rows = experts[e][site][0].shape[0]
        return [pool.submit(_ref_gemm_task, e, site, r0, r1, q, s) for r0, r1 in _row_slices(rows, parts)]

    def join(futs):
        return np.concatenate([f.result() for f in futs], axis=1)

    routed = [(e, np.nonzero((sel == e).any(axis=1))[0]) for e in range(len(experts))]
    routed = [(e, rows) for e, rows in routed if rows.size]
    stage = {}
    for e, rows in routed:  # gate and up of every active expert in flight together
        q, s = np.ascontiguousarray(codes[rows]), np.ascontiguousarray(scales[rows])
        stage[e] = (gemm_jobs(e, 0, q, s), gemm_jobs(e, 1, q, s))
    down = {}
    for e, rows in routed:
        a, b = join(stage[e][0]), join(stage[e][1])
        hc, hs = o.quantize((o.silu(a) * b).astype(np.float32), 4)
        down[e] = gemm_jobs(e, 2, hc, hs)
    dense_w = np.zeros((n, len(experts)), np.float32)
    np.put_along_axis(dense_w, sel, wts.astype(np.float32), axis=1)
    out = np.zeros((n, v.shape[1]), np.float32)
    for e, rows in routed:                  # model.py:391-401, experts ascending
        f = join(down[e])
        out[rows] = out[rows] + dense_w[rows, e, None] * f
    return out


def cpu_reference_steps(n, k, steps, warmup, seed=0):
    """Seconds per full layer (mean over `steps` after `warmup`) and the cores used."""
    import concurrent.futures as cf
    import multiprocessing as mp
    global _REF_EXPERTS
    cores = os.cpu_count() or 1
    v, w, _REF_EXPERTS = host_layer(seed, n)
    times = []
    with cf.ProcessPoolExecutor(max_workers=cores, mp_context=mp.get_context("fork")) as pool:
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            cpu_reference_layer(v, w, _REF_EXPERTS, k, pool, cores)
            if i >= warmup:
                times.append(time.perf_counter() - t0)
    return float(np.mean(times)), cores


def _ref_sample(n, E):
    return (f"the full composed layer every step: batch {n}, all {E} experts, all rows (reference "
            f"_core.lut_gemm_f32 + _core.matmul_f32 from oracle/_ref; output-row slices on one worker "
            f"process per host core)")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    oracle.ref_core()
    n, k, E = args.batch, CFG["top_k"], CFG["n_experts"]
    sec, threads = cpu_reference_steps(n, k, args.steps, args.warmup, args.seed)
    value = n / sec
    emit({
        "impl": "reference", "metric": "MoE-layer tokens/s", "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": CFG["name"], "d_model": CFG["d_model"], "d_ff": CFG["d_ff"],
                   "n_experts": E, "top_k": k, "group_size": CFG["group_size"] or "d_in", "batch": n},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "reference",
                         "sample": _ref_sample(n, E)},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })


def cpu_baseline(n, k, threads=None) -> dict:
    """The GPU arm's cpu_baseline: 3 full layers after 1 warm-up."""
    import oracle
    oracle.ref_core()
    sec, threads = cpu_reference_steps(n, k, 3, 1, seed=1)
    return {"value": n / sec, "unit": "tokens/s", "cores": threads, "kind": "reference",
            "sample": _ref_sample(n, CFG["n_experts"]) + "; 3 layers after 1 warm-up"}


# ---------------------------------------------------------------------------
# GPU side.


def profile_expert_stage(layer, codes_perm, scales_perm, offsets, R, iters):
    """Per-stage device times of the grouped expert stage on the current
    stream (cq_moe_profile_experts records CUDA events between the kernels:
    gate|up GEMM | silu*up + re-quantize | down GEMM), averaged over iters.
    Returns (active experts, algorithmic bytes, (gu_ms, rq_ms, dn_ms))."""
    import ctypes
    import torch
    from paper_2604_10496_b200 import _lib as L
    off = offsets.cpu().numpy()
    n_active = int((np.diff(off) > 0).sum())
    live = int(off[-1])                     # R is the row bound; bytes count the live rows
    desc = layer.desc()
    buf, _ = layer.workspace(max(1, -(-R // layer.top_k)))
    stage_ms = (ctypes.c_float * 3)()
    fexp = torch.empty((max(R, 1), layer.d_model), dtype=torch.float32, device="cuda")
    L.check(L.lib().cq_moe_profile_experts(ctypes.byref(desc), codes_perm.data_ptr(), scales_perm.data_ptr(),
                                            offsets.data_ptr(), R, fexp.data_ptr(), buf.data_ptr(), buf.numel(),
                                            iters, stage_ms, L.stream()))
    return n_active, layer_bytes(n_active, live), tuple(float(x) for x in stage_ms)


def traffic_for(layout):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(f"{layout}:gate_up")
    except (OSError, ValueError):
        return None


def e2e_pipelined(step, x_host, y_host, like, out_shape, stream, steps, barrier, graph=True):
    """Mean device ms per step of: H2D copy of the step's input (pinned) ->
    step(x_dev, out) captured as a CUDA graph -> D2H read of its output, with
    the copies on separate streams and two buffer sets, so copies of adjacent
    steps overlap the compute of this one.  `step` may be a pair, one per buffer
    set (steps with their own internal buffers, e.g. the EP step).  graph=False:
    the steps run eagerly (a step with a host read, e.g. compact EP sizing)."""
    fns = step if isinstance(step, (list, tuple)) else (step, step)
    import torch
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    x_dev = [torch.empty_like(like) for _ in range(2)]
    outs = [torch.empty(out_shape, dtype=torch.float32, device="cuda") for _ in range(2)]
    graphs = []
    with torch.cuda.stream(stream):
        for b in range(2):
            x_dev[b].copy_(x_host)
            fns[b](x_dev[b], outs[b])
            if graph:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    fns[b](x_dev[b], outs[b])
                graphs.append(g.replay)
            else:
                graphs.append(lambda b=b: fns[b](x_dev[b], outs[b]))
    torch.cuda.synchronize()
    ev = lambda: torch.cuda.Event(enable_timing=False)  # noqa: E731
    in_ready, done, out_read = [ev(), ev()], [ev(), ev()], [ev(), ev()]

    def run(k):
        for i in range(k):
            b = i & 1
            with torch.cuda.stream(h2d):
                if i >= 2:
                    h2d.wait_event(done[b])          # step i-2 finished reading x_dev[b]
                x_dev[b].copy_(x_host, non_blocking=True)
                in_ready[b].record(h2d)
            with torch.cuda.stream(stream):
                stream.wait_event(in_ready[b])
                if i >= 2:
                    stream.wait_event(out_read[b])   # step i-2's output was read back
                graphs[b]()
                done[b].record(stream)
            with torch.cuda.stream(d2h):
                d2h.wait_event(done[b])
                y_host[b].copy_(outs[b], non_blocking=True)
                out_read[b].record(d2h)

    run(4)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h2d.wait_event(e0)
    run(steps)
    for b in range(2):  # the last two steps' read-backs
        stream.wait_event(out_read[b])
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


def run_ep(args, rank, world, local):
    """N > 1: expert parallelism (ep.EPStep).  Every rank holds
    E/N experts (identical seeded weights on all ranks, sliced), the router
    weight and any shared experts, and its own tokens.  A step: route ->
    dispatch rows (one per (token, peer), codes as nibbles) -> all_to_all ->
    grouped experts -> per-row partial sums -> all_to_all back -> combine (+
    shared experts, run while the dispatch is in flight).

    Decode configs (MX default, weak scaling: B tokens per rank): fixed-capacity
    rows, no host read, the whole step (both NCCL exchanges) in one CUDA graph.
    Prefill configs (PH/QW/DS, strong scaling: the config's batch split over
    the ranks): counts-first all_to_all-v with exact splits, two micro-batches
    so one batch's exchanges overlap the other's experts, eager."""
    import torch
    import torch.distributed as dist
    from paper_2604_10496_b200 import _lib as L
    from paper_2604_10496_b200.ep import EPStep, expert_range
    from paper_2604_10496_b200.moe import ExpertStack, MoELayer
    from paper_2604_10496_b200.synthetic import moe_inputs_device

    prefill = CFG["batch"] >= 1024
    d, ff, E, k, g = CFG["d_model"], CFG["d_ff"], CFG["n_experts"], CFG["top_k"], CFG["group_size"]
    n = max(1, args.batch // world) if prefill and not args.batch_given else args.batch
    n_sh = CFG.get("n_shared", 0)
    _, w, sites, sh_sites = moe_inputs_device(args.seed, 1, d, ff, E, g, n_shared=n_sh, kc=CFG.get("kc", 16))
    begin, per = expert_range(E, world, rank)
    stacks = [ExpertStack(sites[s][0][begin:begin + per].contiguous(), sites[s][1][begin:begin + per].contiguous(),
                          sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    shared = (tuple(ExpertStack(sh_sites[s][0], sh_sites[s][1], sh_sites[s][2], sh_sites[s][3], g)
                    for s in ("gate", "up", "down")) if n_sh else None)
    del sites
    torch.cuda.empty_cache()
    rotation = None
    if CFG.get("rotation"):
        gen = torch.Generator(device="cuda")
        gen.manual_seed(args.seed + 99)
        rotation = torch.linalg.qr(torch.randn((d, d), generator=gen, device="cuda"))[0].contiguous()
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, rotation=rotation, shared=shared, path=args.path,
                                 expert_begin=begin, n_experts=E)
    if args.path in ("auto", "tc"):
        layer.prepare_tc(layout=args.layout)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(args.seed + 1000 + rank)
    v = torch.randn((n, d), generator=gen, device="cuda").to(torch.bfloat16)
    sizing, mb = ("compact", 2) if prefill else ("fixed", 1)
    step = EPStep(layer, n, rank, world, sizing=sizing, micro_batches=mb)
    stream = torch.cuda.Stream()

    def barrier():
        dist.barrier()
        torch.cuda.synchronize()

    with torch.cuda.stream(stream):
        c0 = L.launch_count()
        step(v)
        launches_per_step = L.launch_count() - c0
        for _ in range(2):
            step(v)
    torch.cuda.synchronize()
    graph, capture_err = None, None
    if sizing == "fixed":  # one step (both NCCL exchanges included) in a CUDA graph; eager if refused
        try:
            g_ = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_, stream=stream):
                step(v)
            graph = g_
        except Exception as exc:
            capture_err = repr(exc)[:200]
            torch.cuda.synchronize()
    run = graph.replay if graph is not None else (lambda: step(v))
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            run()
    torch.cuda.synchronize()

    def timed(fn, steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            barrier()
            e0.record(stream)
            for _ in range(steps):
                fn()
            e1.record(stream)
            e1.synchronize()
            barrier()
        t = torch.tensor([e0.elapsed_time(e1) / steps], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    with ClockSampler(local) as clk:
        ms = timed(run, args.steps)
    xb = step.exchange_bytes()
    xbt = torch.tensor([xb["out"], xb["back"]], dtype=torch.float64, device="cuda")
    dist.all_reduce(xbt, op=dist.ReduceOp.MAX)

    # exposed communication: the same step with both payload exchanges replaced by no-ops (the
    # receive buffers keep the last real step's rows, so the compute is identical), eager, max over ranks
    real_x = step.xchg
    step.xchg = lambda *a: None
    ms_nocomm = timed(lambda: step(v), max(3, min(args.steps, 20)))
    step.xchg = real_x
    ms_eager = timed(lambda: step(v), max(3, min(args.steps, 20)))

    # end to end: pinned H2D -> EP step (both exchanges) -> D2H each step, pipelined as on one GPU
    x_host = v.cpu().pin_memory()
    y_host = [torch.empty((n, d), dtype=torch.float32).pin_memory() for _ in range(2)]
    steps2 = [EPStep(layer, n, rank, world, sizing=sizing, micro_batches=mb) for _ in range(2)]
    e2e_ms = e2e_pipelined([lambda xd, o, st=st: st(xd, out=o) for st in steps2], x_host, y_host, v, (n, d),
                           stream, args.steps, barrier, graph=sizing == "fixed")
    t = torch.tensor([e2e_ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())

    with torch.cuda.stream(stream):
        step(v)
        routes = int(step.offsets[-1].item())   # last micro-batch's grouped routes (profiling input)
        n_active, byt, (gu_ms, rq_ms, dn_ms) = profile_expert_stage(layer, step.codes_perm, step.scales_perm,
                                                                    step.offsets, max(routes, 1),
                                                                    max(3, args.steps))
    pk = peaks()
    tensor_bound = routes >= 128 * max(n_active, 1)
    if tensor_bound:
        achieved, peak_v, unit = 4.0 * routes * d * ff / (gu_ms * 1e-3) / 1e12, pk["bf16_tflops"], "TFLOP/s"
    else:
        achieved, peak_v, unit = byt["gate_up"] / (gu_ms * 1e-3) / 1e9, pk["hbm_gbs"], "GB/s"
    if rank == 0:
        total = n * world
        res = {
            "metric": "MoE-layer tokens/s", "value": total / (ms * 1e-3), "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong" if prefill else "weak", "vs_baseline": None,
            "dtype": "int8/f32", "data": "synthetic (random-init 4-bit codebook weights, N(0,1) bf16 activations)",
            "config": {"workload": CFG["name"], "d_model": d, "d_ff": ff, "n_experts": E, "top_k": k,
                       "n_shared": n_sh, "group_size": g or "d_in", "batch_per_rank": n, "global_batch": total,
                       "parallelism": f"ep{world}", "experts_per_rank": per, "path": args.path,
                       "layout": args.layout, "l2": "weights > L2, no flush needed",
                       "cuda_graph": graph is not None, "ep_rows": "dedup (one row per token and peer)",
                       "ep_sizing": sizing, "micro_batches": mb,
                       **({"capture_error": capture_err} if capture_err else {})},
            "e2e": {"value": total / (e2e_ms * 1e-3), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(x_host.numel() * x_host.element_size()),
                    "d2h_bytes_per_step": int(y_host[0].numel() * y_host[0].element_size()),
                    "pipelined": "H2D / EP step / D2H on three streams, double-buffered"},
            "roofline": {"bound": "tensor" if tensor_bound else "hbm",
                         "kernel": "rank 0's grouped gate|up LUT GEMM (lut_umma_kernel)",
                         "achieved": achieved, "peak": peak_v, "unit": unit, "frac": achieved / peak_v,
                         "peak_src": pk["src"], "traffic": None, "algorithmic_bytes": byt["gate_up"],
                         "kernel_ms": gu_ms, "routes_profiled": routes, "active_local_experts": n_active,
                         "stage_ms": {"gate_up": gu_ms, "silu_requant": rq_ms, "down": dn_ms}},
            "clocks": clk.summary(),
            "gpu_launches": int(launches_per_step * args.steps),
            "ep": {"step_ms_eager": round(ms_eager, 4), "step_ms_without_exchanges": round(ms_nocomm, 4),
                   "comm_exposed_ms": round(max(0.0, ms_eager - ms_nocomm), 4),
                   "exchange_bytes_per_rank_max": {"out": int(xbt[0].item()), "back": int(xbt[1].item())},
                   "note": "exposed = eager step - the same step with both payload exchanges as no-ops "
                           "(max over ranks)"},
        }
        emit(res)
    dist.destroy_process_group()


def run_ours(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 or args.ep:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2604_10496_b200 import _lib
    from paper_2604_10496_b200.moe import ExpertStack, MoELayer
    from paper_2604_10496_b200.synthetic import moe_inputs_device

    if (world > 1 and not args.replicas) or args.ep:
        try:
            return run_ep(args, rank, world, local)
        except Exception as exc:  # report replicas rather than nothing, and say why
            print(f"[bench] expert-parallel path failed ({exc!r}); running replicas", file=sys.stderr)
            args.ep_error = repr(exc)
            torch.cuda.empty_cache()

    n, d, ff, E, k, g = args.batch, CFG["d_model"], CFG["d_ff"], CFG["n_experts"], CFG["top_k"], CFG["group_size"]
    n_sh = CFG.get("n_shared", 0)
    v, w, sites, sh_sites = moe_inputs_device(args.seed + 17 * rank, n, d, ff, E, g, n_shared=n_sh,
                                              kc=CFG.get("kc", 16))
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    shared = (tuple(ExpertStack(sh_sites[s][0], sh_sites[s][1], sh_sites[s][2], sh_sites[s][3], g)
                    for s in ("gate", "up", "down")) if n_sh else None)
    rotation = None
    if CFG.get("rotation"):  # random orthogonal R (rotation.py:38-44 draws a QR of a Gaussian)
        gen = torch.Generator(device="cuda")
        gen.manual_seed(args.seed + 99)
        rotation = torch.linalg.qr(torch.randn((d, d), generator=gen, device="cuda"))[0].contiguous()
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, rotation=rotation, shared=shared, path=args.path)
    if args.path in ("auto", "tc"):
        try:
            layer.prepare_tc(layout=args.layout)
        except Exception as exc:  # tensor-core layout not available for this build
            if args.path == "tc":
                raise
            print(f"[bench] tc path unavailable ({exc}); using the fp32 path", file=sys.stderr)
    path_used = args.path
    out = torch.empty((n, d), dtype=torch.float32, device="cuda")
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()

    # launches per step (counted on an eager run), then capture one step in a graph
    with torch.cuda.stream(stream):
        c0 = _lib.launch_count()
        layer(v, out=out)
        launches_per_step = _lib.launch_count() - c0
        for _ in range(2):
            layer(v, out=out)
    stream.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        layer(v, out=out)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            graph.replay()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk, torch.cuda.stream(stream):
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            graph.replay()  # replays on the current (= timed) stream
        ev1.record(stream)
        ev1.synchronize()
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())

    # end to end through the public API: every step copies its input from pinned host memory
    # and reads its result back; the copies run on their own streams, double-buffered, so
    # step i+1's H2D and step i-1's D2H overlap step i's layer (a serving loop's pipeline)
    x_host = v.cpu().pin_memory()
    y_host = [torch.empty((n, d), dtype=torch.float32).pin_memory() for _ in range(2)]
    e2e_ms = e2e_pipelined(lambda xd, o: layer(xd, out=o), x_host, y_host, v, (n, d), stream, args.steps,
                           barrier)
    t = torch.tensor([e2e_ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())

    # dominant kernel: the grouped gate|up LUT GEMM, timed per stage with CUDA
    # events on its stream (cq_moe_profile_experts records events between the
    # expert-stage kernels: gate|up GEMM | silu*up + re-quantize | down GEMM)
    with torch.cuda.stream(stream):
        layer.route(v)  # codes_perm / scales_perm (the tensor-core forward gathers in-kernel)
        tr = layer.trace(n)
        n_active, byt, (gu_ms, rq_ms, dn_ms) = profile_expert_stage(layer, tr["codes_perm"], tr["scales_perm"],
                                                                    tr["offsets"], n * k, max(3, args.steps))
    pk = peaks()
    R = n * k
    # prefill (>= 128 routes per active expert) is tensor-bound: report the gate|up
    # kernel's algorithmic flops (2*R*2*d*ff, digit planes not counted) against the dense bf16 peak
    tensor_bound = R >= 128 * max(n_active, 1)
    if tensor_bound:
        achieved, peak_v, unit = 4.0 * R * d * ff / (gu_ms * 1e-3) / 1e12, pk["bf16_tflops"], "TFLOP/s"
    else:
        achieved, peak_v, unit = byt["gate_up"] / (gu_ms * 1e-3) / 1e9, pk["hbm_gbs"], "GB/s"
    traffic = traffic_for(args.layout) if args.config == "mx" else None

    if rank == 0:
        res = {
            "metric": "MoE-layer tokens/s", "value": n * world / (ms * 1e-3), "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8/f32",
            "data": "synthetic (random-init 4-bit codebook weights, N(0,1) bf16 activations)",
            "config": {"workload": CFG["name"], "d_model": d, "d_ff": ff, "n_experts": E, "top_k": k,
                       "group_size": g or "d_in", "codebook_k": CFG.get("kc", 16), "batch": n,
                       "parallelism": (f"replicas{world}" + (f" (ep failed: {args.ep_error})"
                                                             if getattr(args, "ep_error", None) else ""))
                       if world > 1 else "single",
                       "path": path_used, "layout": args.layout,
                       "l2": "weights > 126 MB L2, no flush needed",
                       "cuda_graph": True, "active_experts": n_active},
            "e2e": {"value": n * world / (e2e_ms * 1e-3), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(x_host.numel() * x_host.element_size()),
                    "d2h_bytes_per_step": int(y_host[0].numel() * y_host[0].element_size()),
                    "pipelined": "H2D / layer / D2H on three streams, double-buffered"},
            "roofline": {"bound": "tensor" if tensor_bound else "hbm",
                         "kernel": "grouped gate|up LUT GEMM (lut_umma_kernel<3>, tcgen05 kind::i8, A from TMEM)",
                         "achieved": achieved, "peak": peak_v, "unit": unit,
                         "frac": achieved / peak_v, "peak_src": pk["src"],
                         "peak_spec": SPEC_BF16_TFLOPS if tensor_bound else SPEC_HBM_GBS,
                         "frac_spec": achieved / (SPEC_BF16_TFLOPS if tensor_bound else SPEC_HBM_GBS),
                         "traffic": traffic, "algorithmic_bytes": byt["gate_up"], "kernel_ms": gu_ms,
                         "bytes_def": "SURVEY 8(d): ids d_out*d_in/2 + fp32 centroids d_out*(d_in/g)*64 per active "
                                      "expert and matrix, + codes/scales in + fp32 outputs",
                         "stage_ms": {"gate_up": gu_ms, "silu_requant": rq_ms, "down": dn_ms},
                         "layer_frac": byt["layer"] / (ms * 1e-3) / 1e9 / pk["hbm_gbs"]},
            "clocks": clk.summary(),
            "gpu_launches": int(launches_per_step * args.steps),
        }
        if not args.no_cpu_baseline and world == 1:
            try:
                res["cpu_baseline"] = cpu_baseline(n, k, os.cpu_count() or 1)
            except Exception as exc:  # oracle/_ref missing on this box
                res["cpu_baseline"] = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference",
                                       "sample": f"unavailable: {exc}"}
        emit(res)
    if world > 1:
        dist.destroy_process_group()


_JSON_FD = None  # the real stdout: libraries (NCCL's banner, ...) write to fd 1, which main() points at stderr


def emit(res: dict) -> None:
    """The one JSON line on stdout."""
    line = (json.dumps(res) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(line.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, line)


def main():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    args = parse()
    CFG.clear()
    CFG.update(dict(CONFIGS[args.config]), group_size=CONFIGS[args.config].get("group_size", 128))
    args.batch_given = args.batch is not None
    if args.batch is None:
        args.batch = CFG["batch"]
    if args.config != "mx":
        args.no_cpu_baseline = True  # the bounded CPU sample is calibrated for the headline config
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
