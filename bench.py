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

N > 1 (torchrun): one independent replica per GPU over its own batch (the
single-GPU layer fits in HBM; the expert-parallel path is ep.py), reported as
weak scaling; time = max over ranks.
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

CFG = dict(name="mixtral-8x7b-moe-layer-decode", d_model=4096, d_ff=14336, n_experts=8, top_k=2,
           group_size=128)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--batch", type=int, default=64)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--path", default="auto", choices=["auto", "tc", "f32", "ordered"])
    p.add_argument("--layout", default="umma128u", choices=["umma128", "umma128u", "mma16"],
                   help="tensor-core weight layout / kernel")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--seed", type=int, default=0)
    return p.parse_args()


def layer_bytes(n_active: int, n: int, k: int) -> dict:
    """Algorithmic HBM bytes: reference-format weights of the
    active experts + activations, per layer and for the gate|up kernel."""
    d, ff, g = CFG["d_model"], CFG["d_ff"], CFG["group_size"]
    w_gu = 2 * (ff * d // 2 + ff * (d // g) * 16 * 4)        # gate + up ids + centroids
    w_dn = d * ff // 2 + d * (ff // g) * 16 * 4
    R = n * k
    gu = n_active * w_gu + R * d + R * 4 + R * ff * 4         # + codes, scales in; hidden out
    dn = n_active * w_dn + R * ff + R * 4 + R * d * 4
    return dict(gate_up=gu, down=dn, layer=gu + dn + d * CFG["n_experts"] * 4)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": p["hbm_gbs"], "src": "measured"}
    except (OSError, KeyError, ValueError):
        return {"hbm_gbs": 6650.0, "src": "fallback"}


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
            mats.append(((rng.standard_normal((do, di // g, 16), dtype=np.float32) / math.sqrt(di)),
                         rng.integers(0, 256, (do, di // 2), dtype=np.uint8), g))
        experts.append(mats)
    return v, w, experts


def cpu_reference_step(v, w, experts, k, threads, expert_sample):
    """The composed MoE block on the reference's native kernels
    (oracle/_ref: _core.matmul_f32 for the router, _core.lut_gemm_f32 with the
    reference's token-block threading for the experts), restricted to one
    sampled expert; returns seconds scaled to the whole layer."""
    import oracle
    from oracle import oracle as o
    t0 = time.perf_counter()
    codes, scales = o.quantize(v, 4)
    core = oracle.ref_core()
    logits = np.zeros((v.shape[0], w.shape[1]), np.float32)
    core.matmul_f32(np.ascontiguousarray(codes.astype(np.float32) * scales[:, None]), w, logits)
    sel, wts = o.select_top_k(logits, k)
    t_route = time.perf_counter() - t0
    E = len(experts)
    t_exp = 0.0
    for e in expert_sample:
        rows = np.nonzero((sel == e).any(axis=1))[0]
        if rows.size == 0:
            continue
        t1 = time.perf_counter()
        bt = max(1, -(-rows.size // threads))
        (cg, ig, gg), (cu, iu, gu), (cd, idn, gd) = experts[e]
        a = oracle.ref_lut_gemm(codes[rows], scales[rows], ig, cg, gg, bt, threads)
        b = oracle.ref_lut_gemm(codes[rows], scales[rows], iu, cu, gu, bt, threads)
        hc, hs = o.quantize((o.silu(a) * b).astype(np.float32), 4)
        oracle.ref_lut_gemm(hc, hs, idn, cd, gd, bt, threads)
        t_exp += time.perf_counter() - t1
    return t_route + t_exp * E / len(expert_sample)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    oracle.ref_core()
    threads = os.cpu_count() or 1
    n, k, E = args.batch, CFG["top_k"], CFG["n_experts"]
    v, w, experts = host_layer(args.seed, n)
    times = []
    for i in range(args.warmup + args.steps):
        t = cpu_reference_step(v, w, experts, k, threads, [i % E])
        if i >= args.warmup:
            times.append(t)
    sec = float(np.mean(times))
    value = n / sec
    sample = (f"batch {n}: router for all tokens, 1 of {E} experts per step (rotating), "
              f"expert time x{E} (per-expert work is additive)")
    print(json.dumps({
        "impl": "reference", "metric": "MoE-layer tokens/s", "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": CFG["name"], "d_model": CFG["d_model"], "d_ff": CFG["d_ff"],
                   "n_experts": E, "top_k": k, "group_size": CFG["group_size"], "batch": n},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def cpu_baseline(n, k, threads) -> dict:
    import oracle
    oracle.ref_core()
    v, w, experts = host_layer(1, n)
    E = CFG["n_experts"]
    times = [cpu_reference_step(v, w, experts, k, threads, [e]) for e in (0, 3, 6)]
    sec = float(np.mean(times))
    return {"value": n / sec, "unit": "tokens/s", "cores": threads, "kind": "reference",
            "sample": f"batch {n}, experts 0/3/6 timed one per step, expert time x{E}; "
                      f"reference _core.lut_gemm_f32 + _core.matmul_f32 (oracle/_ref)"}


# ---------------------------------------------------------------------------
# GPU side.


def run_ours(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2604_10496_b200 import _lib
    from paper_2604_10496_b200.moe import ExpertStack, MoELayer
    from paper_2604_10496_b200.synthetic import moe_inputs_device

    n, d, ff, E, k, g = args.batch, CFG["d_model"], CFG["d_ff"], CFG["n_experts"], CFG["top_k"], CFG["group_size"]
    v, w, sites, _ = moe_inputs_device(args.seed + 17 * rank, n, d, ff, E, g)
    stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=k, path=args.path)
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

    # end to end through the public API: pinned host input -> device -> forward -> host output
    x_host = v.cpu().pin_memory()
    y_host = torch.empty((n, d), dtype=torch.float32).pin_memory()
    with torch.cuda.stream(stream):
        x_dev = torch.empty_like(v)
        for _ in range(3):
            x_dev.copy_(x_host, non_blocking=True)
            layer(x_dev, out=out)
            y_host.copy_(out, non_blocking=True)
        stream.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            x_dev.copy_(x_host, non_blocking=True)
            layer(x_dev, out=out)
            y_host.copy_(out, non_blocking=True)
        e1.record(stream)
        e1.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([e2e_ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())

    # dominant kernel: the grouped gate|up LUT GEMM, timed per stage with CUDA
    # events on its stream (cq_moe_profile_experts records events between the
    # expert-stage kernels: gate|up GEMM | silu*up + re-quantize | down GEMM)
    tr = layer.trace(n)
    offsets = tr["offsets"].cpu().numpy()
    n_active = int((np.diff(offsets) > 0).sum())
    byt = layer_bytes(n_active, n, k)
    from paper_2604_10496_b200 import _lib as L
    import ctypes
    desc = layer.desc()
    buf, _ = layer.workspace(n)
    stage_ms = (ctypes.c_float * 3)()
    with torch.cuda.stream(stream):
        fexp = torch.empty((n * k, d), dtype=torch.float32, device="cuda")
        L.check(L.lib().cq_moe_profile_experts(ctypes.byref(desc), tr["codes_perm"].data_ptr(),
                                                tr["scales_perm"].data_ptr(), tr["offsets"].data_ptr(), n * k,
                                                fexp.data_ptr(), buf.data_ptr(), buf.numel(), max(3, args.steps),
                                                stage_ms, L.stream()))
    gu_ms, rq_ms, dn_ms = (float(x) for x in stage_ms)
    pk = peaks()
    achieved = byt["gate_up"] / (gu_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(f"{args.layout}:gate_up")
    except (OSError, ValueError):
        pass

    if rank == 0:
        res = {
            "metric": "MoE-layer tokens/s", "value": n * world / (ms * 1e-3), "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8/f32",
            "data": "synthetic (random-init 4-bit codebook weights, N(0,1) bf16 activations)",
            "config": {"workload": CFG["name"], "d_model": d, "d_ff": ff, "n_experts": E, "top_k": k,
                       "group_size": g, "batch": n, "parallelism": f"replicas{world}" if world > 1 else "single",
                       "path": path_used, "layout": args.layout, "l2": "weights 1.41 GB > 126 MB L2, no flush needed",
                       "cuda_graph": True, "active_experts": n_active},
            "e2e": {"value": n * world / (e2e_ms * 1e-3), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(x_host.numel() * x_host.element_size()),
                    "d2h_bytes_per_step": int(y_host.numel() * y_host.element_size())},
            "roofline": {"bound": "hbm",
                         "kernel": "grouped gate|up LUT GEMM (lut_umma_kernel<3>, tcgen05 kind::i8, A from TMEM)",
                         "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"], "peak_src": pk["src"],
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
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
