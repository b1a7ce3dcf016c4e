"""Randomized parity sweep of the tensor-core layer (GPU): random shapes, expert
counts, top-k, group sizes, codebook sizes, shared experts (run as extra
segments of the routed launches) and an online rotation (tensor cores + the
certified quantizer); the tcgen05 path against the ordered path (layer
tolerance 1e-2), the two GEMM geometries against each other (bitwise), repeat
calls (bitwise), and with a rotation the codes / scales / top-k against the
ordered rotation's (bitwise).

    python tools/stress_parity.py [n_cases] [seed]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as o  # noqa: E402
from paper_2604_10496_b200.moe import ExpertStack, MoELayer  # noqa: E402
from paper_2604_10496_b200.synthetic import moe_inputs_device  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
worst = 0.0
for i in range(cases):
    E = int(rng.choice([4, 8, 16, 24, 32, 64, 128]))
    k = int(rng.integers(1, min(8, E) + 1))
    d = int(rng.choice([256, 512, 1024, 2048]))
    ff = int(rng.choice([256, 384, 768, 1408 if d >= 1024 else 512]))
    n = int(rng.choice([1, 3, 17, 64, 130, 300, 600]))
    g = int(rng.choice([128, 0]))
    kc = int(rng.choice([16, 16, 8, 4]))
    n_sh = int(rng.choice([0, 0, 1, 2]))
    rot = bool(rng.random() < 0.3) and d % 256 == 0
    v, w, sites, sh = moe_inputs_device(1000 + i, n, d, ff, E, g, kc=kc, n_shared=n_sh)
    st = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
    shared = (tuple(ExpertStack(sh[s][0], sh[s][1], sh[s][2], sh[s][3], g) for s in ("gate", "up", "down"))
              if n_sh else None)
    R = None
    if rot:
        gen = torch.Generator(device="cuda")
        gen.manual_seed(77 + i)
        R = torch.linalg.qr(torch.randn((d, d), generator=gen, device="cuda"))[0].contiguous()
    layer = MoELayer.from_stacks(w, *st, top_k=k, path="tc", shared=shared, rotation=R)
    layer.prepare_tc()
    out = layer(v).clone()
    again = layer(v).clone()
    os.environ["CQ_UMMA_GEOMETRY"] = "decode"
    dec = layer(v).clone()
    os.environ["CQ_UMMA_GEOMETRY"] = "prefill"
    pre = layer(v).clone() if n * k >= 64 else dec
    del os.environ["CQ_UMMA_GEOMETRY"]
    rok = True
    if rot:  # certified codes == the ordered rotation's, so routing matches bit for bit
        tr = {key: t.clone() for key, t in layer.trace(n).items() if key in ("codes", "scales", "selected")}
        layer.exact_rotation = True
        layer(v)
        tro = layer.trace(n)
        rok = all(torch.equal(tr[key], tro[key]) for key in tr)
        layer.exact_rotation = False
    ref = layer(v, path="ordered").clone()
    err = o.relative_error(out.cpu().numpy(), ref.cpu().numpy())
    worst = max(worst, err)
    ok = torch.equal(out, again) and torch.equal(dec, pre) and torch.equal(out, dec) and err <= 1e-2 and rok
    print(f"case {i:2d} n={n:4d} E={E:3d} k={k} d={d:4d} ff={ff:4d} g={g or 'd_in'} K={kc:2d} sh={n_sh} "
          f"rot={int(rot)}: "
          f"rel err {err:.2e} {'ok' if ok else 'FAIL'}", flush=True)
    if not ok:
        sys.exit(1)
print(f"all {cases} cases ok, worst layer error {worst:.2e}")
