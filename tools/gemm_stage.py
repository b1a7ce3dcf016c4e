"""Stage times of the grouped expert GEMMs (gate|up, silu|requant, down) at one
config, for A/B runs of library variants:

    CQ_B200_LIB=paper_2604_10496_b200/libcq_b200_x.so python tools/gemm_stage.py [mx|qw64|ph|qw|ds] [iters]

Prints one line per run: variant, stage µs (CUDA events around each kernel,
cq_moe_profile_experts), gate|up algorithmic GB/s."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
from paper_2604_10496_b200 import _lib  # noqa: E402
from paper_2604_10496_b200.moe import ExpertStack, MoELayer  # noqa: E402
from paper_2604_10496_b200.synthetic import moe_inputs_device  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "mx"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
C = bench.CONFIGS[cfg]
n, d, ff, E, k, g = C["batch"], C["d_model"], C["d_ff"], C["n_experts"], C["top_k"], C.get("group_size", 128)
bench.CFG.clear()
bench.CFG.update(dict(C, group_size=g))
v, w, sites, _ = moe_inputs_device(0, n, d, ff, E, g, kc=C.get("kc", 16))
stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
layer = MoELayer.from_stacks(w, *stacks, top_k=k, path="tc").prepare_tc()
layer.route(v)
tr = layer.trace(n)
bench.profile_expert_stage(layer, tr["codes_perm"], tr["scales_perm"], tr["offsets"], n * k, 2)  # warm-up
n_active, byt, (gu, rq, dn) = bench.profile_expert_stage(layer, tr["codes_perm"], tr["scales_perm"], tr["offsets"],
                                                          n * k, iters)
print(f"{os.path.basename(_lib.LIB_PATH)} {cfg}: gate|up {gu * 1e3:.1f} us ({byt['gate_up'] / gu / 1e6:.0f} GB/s), "
      f"silu|requant {rq * 1e3:.1f} us, down {dn * 1e3:.1f} us ({byt['down'] / dn / 1e6:.0f} GB/s)", flush=True)
