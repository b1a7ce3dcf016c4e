"""Warm device time of the routing stage (cq_moe_route: quantize, router
logits, top-k, permutation, gather) replayed as a CUDA graph, over d_model, so
the slope gives the router chain's cost per column.

    python tools/route_bench.py [n] [E] [d ...]
"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_10496_b200 import _lib  # noqa: E402
from paper_2604_10496_b200.moe import ExpertStack, MoELayer  # noqa: E402
from paper_2604_10496_b200.synthetic import moe_inputs_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
E = int(sys.argv[2]) if len(sys.argv) > 2 else 8
L = _lib.lib()
s = torch.cuda.Stream()
for d in ([int(a) for a in sys.argv[3:]] or (1024, 2048, 4096, 8192)):
    v, w, sites, _ = moe_inputs_device(0, n, d, 128, E, 128)
    stacks = [ExpertStack(sites[x][0], sites[x][1], sites[x][2], sites[x][3], 128) for x in ("gate", "up", "down")]
    layer = MoELayer.from_stacks(w, *stacks, top_k=2, path="f32")
    layer(v)
    buf, _ = layer.workspace(n)
    dsc = layer.desc()

    def route():
        _lib.check(L.cq_moe_route(ctypes.byref(dsc), v.data_ptr(), _lib.dtype_code(v), n, buf.data_ptr(),
                                  buf.numel(), _lib.stream()))

    with torch.cuda.stream(s):
        route()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                route()
        for _ in range(3):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(10):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    print(f"n={n} E={E} d={d}: route {e0.elapsed_time(e1) / 200 * 1e3:.2f} us")
