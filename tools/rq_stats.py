"""Task statistics of the certified rotation quantizer at the PH bench workload: recomputed chains
per row (status[2]) and their spread over columns (from the tensor-core v and the pick rule).
GPU only:  python tools/rq_stats.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
from paper_2604_10496_b200 import _lib  # noqa: E402
from paper_2604_10496_b200.moe import ExpertStack, MoELayer  # noqa: E402
from paper_2604_10496_b200.synthetic import moe_inputs_device  # noqa: E402

C = bench.CONFIGS["ph"]
n, d, ff, E, k, g = C["batch"], C["d_model"], C["d_ff"], C["n_experts"], C["top_k"], 128
v, w, sites, _ = moe_inputs_device(0, n, d, ff, E, g)
gen = torch.Generator(device="cuda")
gen.manual_seed(1234)
R = torch.linalg.qr(torch.randn((d, d), generator=gen, device="cuda"))[0].contiguous()
stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
layer = MoELayer.from_stacks(w, *stacks, top_k=k, rotation=R, path="tc").prepare_tc()
buf, offs = layer.workspace(n)
st = offs[_lib.WS_NAMES.index("status")]
buf[st:st + 16].zero_()
layer(v)
torch.cuda.synchronize()
status = buf[st:st + 16].view(torch.int32).cpu()
print("recomputed chains", int(status[2]), "per row", int(status[2]) / n)
vt = buf[offs[_lib.WS_NAMES.index("rotated")]:].view(torch.float32)[:n * d].view(n, d)
mx = vt.abs().amax(1, keepdim=True)
cand = vt.abs() >= mx * (1 - 3e-4)
print("max candidates per row", cand.sum(1).float().mean().item())
cols = cand.sum(0)
print("candidate columns: max per column", cols.max().item(), "columns used", (cols > 0).sum().item())
top = torch.topk(cols, 5)
print("top columns", top.indices.tolist(), top.values.tolist())
