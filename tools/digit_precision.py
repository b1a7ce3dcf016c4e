"""Layer error of integer-digit weights of a given width, emulated on the fp32
path: centroids rounded to m = rint(c / s_row) * s_row with s_row = max|c| of
the row / (2^(bits-1) - 1), then the fp32 CUDA-core layer against the ordered
layer on the original centroids (Mixtral shape, decode batch 64).  14 bits is
two 7-bit digit planes, 21 bits three (the shipped gate|up layout), 16 bits a
u8 low / s8 high two-plane layout.  GPU only.

    python tools/digit_precision.py
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_10496_b200.moe import ExpertStack, MoELayer  # noqa: E402
from paper_2604_10496_b200.synthetic import moe_inputs_device  # noqa: E402

n, d, ff, E, k, g = 64, 4096, 14336, 8, 2, 128
v, w, sites, _ = moe_inputs_device(0, n, d, ff, E, g)


def stacks(round_bits=None, round_down=None):
    out = []
    for s in ("gate", "up", "down"):
        ids, cents, di, do = sites[s]
        bits = round_down if s == "down" else round_bits
        if bits:
            c = cents.view(E, do, -1)
            sc = c.abs().amax(dim=2, keepdim=True) / float(2 ** (bits - 1) - 1)
            sc = torch.where(sc > 0, sc, torch.ones_like(sc))
            cents = (torch.round(c / sc) * sc).view_as(cents).contiguous()
        out.append(ExpertStack(ids, cents, di, do, g))
    return out


ref_layer = MoELayer.from_stacks(w, *stacks(), top_k=k, path="ordered")
ref = ref_layer(v, path="ordered").clone()


def err(x):
    dif = (x - ref).abs()
    return dif.max().item() / ref.abs().max().item(), (torch.linalg.norm(x - ref) / torch.linalg.norm(ref)).item()


print("f32 path, fp32 centroids", err(MoELayer.from_stacks(w, *stacks(), top_k=k, path="f32")(v).clone()))
for gu, dn in [(21, 14), (16, 14), (16, 16), (15, 14), (14, 14), (18, 14)]:
    layer = MoELayer.from_stacks(w, *stacks(gu, dn), top_k=k, path="f32")
    print(f"gate/up {gu}-bit, down {dn}-bit", err(layer(v).clone()))
