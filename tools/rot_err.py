"""Error of the tcgen05 rotation against the reference's ordered chain (the
fp32 v = x @ R of pipeline.py:516), per element relative to the row's max|v|:
the distribution that sizes the certified quantizer's recompute band."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
from paper_2604_10496_b200 import _lib  # noqa: E402
from test_gpu_configs import _build  # noqa: E402


def rotated(layer, n, d):
    buf, offs = layer.workspace(n)
    o = offs[_lib.WS_NAMES.index("rotated")]
    return buf[o:o + n * d * 4].view(torch.float32).view(n, d).clone()


for seed in (107, 108, 109):
    c, x, layer, host = _build("ph", seed, rotation=True)
    n, d = c["n"], c["d"]
    layer(x)
    v_tc = rotated(layer, n, d)
    s_tc = layer.trace(n)["scales"].clone()
    layer.exact_rotation = True
    layer(x)
    v_ch = rotated(layer, n, d)
    s_ch = layer.trace(n)["scales"].clone()
    mx = v_ch.abs().amax(1, keepdim=True)
    rel = ((v_tc - v_ch).abs() / mx).flatten()
    q = torch.quantile(rel[torch.randperm(rel.numel(), device=rel.device)[:4_000_000]], torch.tensor(
        [0.5, 0.99, 0.9999], device=rel.device))
    emax = float(rel.max())
    s = s_ch.view(-1, 1)
    frac = {}
    for kappa in (4, 16, 64):
        eps = kappa * emax * mx
        t = v_tc / s
        dist = (t - torch.floor(t) - 0.5).abs()          # distance of v/s to the nearest .5 boundary
        frac[kappa] = float((dist * s < eps).float().mean())
    print(f"seed {seed}: |v_tc - v_chain| / row max: median {q[0]:.2e} p99 {q[1]:.2e} p99.99 {q[2]:.2e} "
          f"max {emax:.2e}; scales differ on {(s_tc != s_ch).float().mean():.3f} of rows; "
          f"flagged fraction at kappa x max: {frac}", flush=True)
