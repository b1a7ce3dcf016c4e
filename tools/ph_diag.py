"""PH (rotation) diagnostics: per-token error of the tcgen05 path against the
bit-exact path, split by whether the tcgen05 rotation moved any A4 code of the
token, and the same with the exact rotation on the tcgen05 GEMMs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import oracle  # noqa: E402
from oracle import oracle as o  # noqa: E402
from test_gpu_configs import _build  # noqa: E402

c, x, layer, host = _build("ph", 107, rotation=True)
tc = layer(x).clone().cpu().numpy()
tr = {k: t.cpu().numpy().copy() for k, t in layer.trace(c["n"]).items()}
layer.exact_rotation = True
tc_exact_rot = layer(x).clone().cpu().numpy()
tr2 = {k: t.cpu().numpy().copy() for k, t in layer.trace(c["n"]).items()}
exact = layer(x, path="ordered").cpu().numpy()
moved = (tr["codes"] != tr2["codes"]).any(1)
flip = (np.sort(tr["selected"], 1) != np.sort(tr2["selected"], 1)).any(1)


def tokerr(a, b):
    return np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)


for name, got in (("tc rotation + tc GEMMs", tc), ("exact rotation + tc GEMMs", tc_exact_rot)):
    e = tokerr(got, exact)
    print(f"{name}: Frobenius {o.relative_error(got, exact):.2e}; tokens moved {moved.sum()} flipped {flip.sum()}")
    for lab, m in (("unmoved", ~moved), ("moved, same routing", moved & ~flip), ("flipped", flip)):
        if m.any():
            print(f"   {lab:22s} n={m.sum():5d} Frobenius {o.relative_error(got[m], exact[m]):.2e} "
                  f"max token {e[m].max():.2e} p99 {np.quantile(e[m], 0.99):.2e}")
    idx = np.argsort(-e)[:8]
    print("   worst tokens:", [(int(t), f"{e[t]:.2e}", bool(moved[t]), bool(flip[t])) for t in idx])
for t in np.nonzero(moved & ~flip)[0][:6]:
    d = np.nonzero(tr["codes"][t] != tr2["codes"][t])[0]
    print(f"token {t}: {d.size} codes differ, scale tc/exact {tr['scales'][t]:.9e}/{tr2['scales'][t]:.9e}, "
          f"first diffs {[(int(j), int(tr['codes'][t, j]), int(tr2['codes'][t, j])) for j in d[:6]]}, "
          f"selected {tr['selected'][t]} / {tr2['selected'][t]}, weights {tr['weights'][t]} / {tr2['weights'][t]}")
