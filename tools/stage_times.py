"""Warm per-stage device times of one MoE layer step (each stage captured in its
own CUDA graph and replayed), to see where a decode step's time goes."""
import ctypes, sys
import torch
sys.path.insert(0, ".")
from paper_2604_10496_b200 import _lib
from paper_2604_10496_b200.moe import ExpertStack, MoELayer
from paper_2604_10496_b200.synthetic import moe_inputs_device

n, d, ff, E, k, g = 64, 4096, 14336, 8, 2, 128
v, w, sites, _ = moe_inputs_device(0, n, d, ff, E, g)
stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
layer = MoELayer.from_stacks(w, *stacks, top_k=k, path="tc")
layer.prepare_tc()
out = torch.empty((n, d), device="cuda")
layer(v, out=out)
buf, _ = layer.workspace(n)
dsc = layer.desc()
layer.route(v)  # codes_perm (the tensor-core forward gathers in-kernel)
tr = layer.trace(n)
L = _lib.lib()
fexp = torch.empty((n * k, d), device="cuda")

def route():
    _lib.check(L.cq_moe_route(ctypes.byref(dsc), v.data_ptr(), _lib.dtype_code(v), n, buf.data_ptr(), buf.numel(), _lib.stream()))
def experts():
    _lib.check(L.cq_moe_experts(ctypes.byref(dsc), tr["codes_perm"].data_ptr(), tr["scales_perm"].data_ptr(), tr["offsets"].data_ptr(), n * k, fexp.data_ptr(), buf.data_ptr(), buf.numel(), _lib.stream()))
def combine():
    _lib.check(L.cq_moe_combine(tr["selected"].data_ptr(), tr["weights"].data_ptr(), tr["inv"].data_ptr(), tr["fout"].data_ptr(), n, k, d, None, 0, out.data_ptr(), _lib.stream()))
def full():
    layer(v, out=out)

s = torch.cuda.Stream()
for name, fn in (("route", route), ("experts", experts), ("combine", combine), ("full", full)):
    with torch.cuda.stream(s):
        fn(); fn()
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=s):
            fn()
        for _ in range(5): gph.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(200): gph.replay()
        e1.record(s)
    torch.cuda.synchronize()
    print(f"{name:8s} {e0.elapsed_time(e1) / 200 * 1000:8.1f} us")
