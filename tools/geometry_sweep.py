"""Decode (32-token passes) vs prefill (128-token passes) geometry of the
tcgen05 LUT GEMM on one expert's gate|up shape, over the routed row count
(expert parallelism grows rows per expert with the GPU count).  CQ_UMMA_GEOMETRY=decode|prefill
forces one geometry; run once with each and once without.

    python tools/geometry_sweep.py [d_in d_out]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_10496_b200 import QuantizedActivations, lut_gemm_tc  # noqa: E402
from paper_2604_10496_b200.lutgemm import PackedClusteredWeights  # noqa: E402

d_in, d_out = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (4096, 28672)
gen = torch.Generator(device="cuda")
gen.manual_seed(0)
cent = torch.randn((d_out, d_in // 128, 16), generator=gen, device="cuda") / 64.0
ids = torch.randint(0, 256, (d_out, d_in // 2), generator=gen, device="cuda", dtype=torch.int32).to(torch.uint8)
pw = PackedClusteredWeights(cent, ids, d_in, 128)
pw.prepare_tc(3, "umma128u")
s = torch.cuda.Stream()
for n in (32, 64, 96, 128, 192, 256, 384):
    qa = QuantizedActivations(torch.randint(-8, 8, (n, d_in), generator=gen, device="cuda", dtype=torch.int8),
                              torch.rand((n,), generator=gen, device="cuda") + 0.5, 4)
    with torch.cuda.stream(s):
        lut_gemm_tc(qa, pw, 3, "umma128u")
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            lut_gemm_tc(qa, pw, 3, "umma128u")
        for _ in range(3):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(20):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    print(f"n={n}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
