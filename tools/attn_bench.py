"""Attention-site LUT GEMMs at decode sizes: one q|k|v launch vs three, and the
out projection (d x d sites, g = 128), timed as CUDA graphs with CUDA events.
Reports algorithmic GB/s (ids d*d/2 + fp32 centroids d*(d/g)*64
per site) against the measured HBM peak.

    python tools/attn_bench.py [d]
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_10496_b200 import lut_gemm_tc, quantize_activations  # noqa: E402
from paper_2604_10496_b200.attention import OutLinear, QKVLinear  # noqa: E402
from paper_2604_10496_b200.lutgemm import PackedClusteredWeights  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
g = 128
peak = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6548.8) if len(sys.argv) < 3 else float(sys.argv[2])
gen = torch.Generator(device="cuda")
gen.manual_seed(0)


def site():
    c = torch.randn((d, d // g, 16), generator=gen, device="cuda") / float(np.sqrt(d))
    i = torch.randint(0, 256, (d, d // 2), generator=gen, device="cuda", dtype=torch.int32).to(torch.uint8)
    return PackedClusteredWeights(c, i, d, g)


pws = [site() for _ in range(4)]
qkv = QKVLinear(*pws[:3])
outp = OutLinear(pws[3])
for pw in pws[:3]:
    pw.prepare_tc(3, "umma128u")
site_bytes = d * d // 2 + d * (d // g) * 64
s = torch.cuda.Stream()


def timed(fn, reps=50):
    with torch.cuda.stream(s):
        fn()
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=s):
            fn()
        for _ in range(5):
            gph.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            gph.replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


for n in (1, 8, 64):
    x = torch.randn((n, d), generator=gen, device="cuda").to(torch.bfloat16)
    qa = quantize_activations(x, check_finite=False)
    t_f = timed(lambda: lut_gemm_tc(qa, qkv.w, 3, "umma128u"))
    t_s = timed(lambda: [lut_gemm_tc(qa, pw, 3, "umma128u") for pw in pws[:3]])
    t_o = timed(lambda: lut_gemm_tc(qa, outp.w, 3, "umma128u"))
    gbs = 3 * site_bytes / (t_f * 1e-6) / 1e9
    print(f"d={d} n={n}: q|k|v one launch {t_f:.1f} us ({gbs:.0f} GB/s, {gbs / peak:.2f} of HBM) | "
          f"three launches {t_s:.1f} us | out {t_o:.1f} us ({site_bytes / (t_o * 1e-6) / 1e9:.0f} GB/s)")
