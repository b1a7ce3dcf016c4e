"""Layer error of the tensor-core path vs the bit-exact ordered path for digit-plane
configurations (Mixtral layer shape, decode batch 64).  Prints max-abs and Frobenius
relative errors.  GPU only; used to choose the default."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2604_10496_b200.moe import ExpertStack, MoELayer
from paper_2604_10496_b200.synthetic import moe_inputs_device

n, d, ff, E, k, g = 64, 4096, 14336, 8, 2, 128
v, w, sites, _ = moe_inputs_device(0, n, d, ff, E, g)
stacks = [ExpertStack(sites[s][0], sites[s][1], sites[s][2], sites[s][3], g) for s in ("gate", "up", "down")]
layer = MoELayer.from_stacks(w, *stacks, top_k=k, path="ordered")
ref = layer(v, path="ordered").clone()
f32 = layer(v, path="f32").clone()

def err(x):
    dif = (x - ref).abs()
    return dif.max().item() / ref.abs().max().item(), (torch.linalg.norm(x - ref) / torch.linalg.norm(ref)).item()

print("f32 path", err(f32))
for pgu, pdn, lay in [(3, 2, "umma128u"), (3, 3, "umma128u"), (2, 2, "umma128u")]:
    layer.prepare_tc(pgu, pdn, layout=lay)
    out = layer(v, path="tc").clone()
    print(f"tc planes gate/up={pgu} down={pdn} {lay}", err(out))
