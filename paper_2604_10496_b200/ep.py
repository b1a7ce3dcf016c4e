"""Expert parallelism for the MoE layer: experts sharded
over the ranks of one node, tokens data-parallel at the input, one exchange
each way over NCCL.

Per rank, one forward pass:
  1. route its own tokens: A4 codes + scales, ordered router logits, top-k
     (bit-exact; `cq_moe_route`);
  2. dispatch: every (token, slot) route goes to the rank owning its expert
     (experts [r*E/G, (r+1)*E/G) live on rank r).  Counts go first
     (all_to_all of G ints), then the payload: the token's int8 codes (exact —
     quantization is per token and happens before routing, model.py:379), its
     fp32 scale and the local expert id (all_to_all_single with the counts as
     split sizes);
  3. the owner regroups the received rows by local expert (stable) and runs the
     grouped gate|up -> silu*up -> re-quantize -> down stage (`cq_moe_experts`);
  4. return: the per-route fp32 outputs travel back by the inverse split;
  5. combine on the source rank in ascending expert order (`cq_moe_combine`),
     so the result is identical to the single-GPU layer.

The compute steps are pluggable: `CudaBackend` (libcq_b200.so) or
`OracleBackend` (the CPU oracle, used by the world_size-2 gloo tests of this
host logic).  Deduplication of a token routed to two experts of one rank is
not done yet: each route carries its own copy of the codes (d bytes + 8).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib


def expert_range(n_experts: int, world: int, rank: int) -> tuple[int, int]:
    if n_experts % world:
        raise ValueError(f"{n_experts} experts do not split over {world} ranks")
    per = n_experts // world
    return rank * per, per


def plan_dispatch(selected: torch.Tensor, n_experts: int, world: int):
    """Route -> destination bookkeeping (pure index work, any device).

    Returns order (routes sorted by destination rank, stable in (t, slot)
    order), the destination of each sorted route, and per-rank send counts."""
    per = n_experts // world
    flat_e = selected.reshape(-1).long()
    dest = flat_e // per
    order = torch.sort(dest, stable=True).indices
    counts = torch.bincount(dest, minlength=world)
    return order, dest[order], counts


def all_to_all_counts(send_counts: torch.Tensor, group=None) -> torch.Tensor:
    recv = torch.empty_like(send_counts)
    dist.all_to_all_single(recv, send_counts, group=group)
    return recv


def exchange(t: torch.Tensor, send_counts: list, recv_counts: list, group=None) -> torch.Tensor:
    out = torch.empty((sum(recv_counts),) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    dist.all_to_all_single(out, t.contiguous(), output_split_sizes=recv_counts, input_split_sizes=send_counts,
                           group=group)
    return out


class EPMoE:
    """One rank's share of an expert-parallel MoE layer."""

    def __init__(self, backend, n_experts: int, top_k: int, rank: int, world: int, group=None):
        self.be, self.E, self.k, self.rank, self.world, self.group = backend, n_experts, top_k, rank, world, group
        self.begin, self.per = expert_range(n_experts, world, rank)

    # The three local phases; `forward` puts the two exchanges between them.
    def dispatch(self, x: torch.Tensor) -> dict:
        """Route the rank's tokens and build the send buffers, ordered by
        destination rank (stable in (token, slot) order)."""
        codes, scales, selected, weights = self.be.route(x)
        order, _, send = plan_dispatch(selected, self.E, self.world)
        tok = order // self.k
        eid = (selected.reshape(-1).long()[order] % self.per).to(torch.int32)
        return {"selected": selected, "weights": weights, "order": order, "send": send,
                "codes": codes[tok], "scales": scales[tok], "eid": eid}

    def compute(self, r_codes, r_scales, r_eid) -> torch.Tensor:
        """Received routes -> per-route fp32 expert outputs, in received order."""
        return self.be.experts(r_codes, r_scales, r_eid, self.per)

    def finish(self, st: dict, f_back: torch.Tensor) -> torch.Tensor:
        """Returned outputs (rows in send order) -> combined moe_sum."""
        f_routes = torch.empty_like(f_back)
        f_routes[st["order"]] = f_back                                    # (t, slot) order
        return self.be.combine(st["selected"], st["weights"], f_routes)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        st = self.dispatch(x)
        recv = all_to_all_counts(st["send"], self.group)
        send_l, recv_l = st["send"].tolist(), recv.tolist()
        r_codes = exchange(st["codes"], send_l, recv_l, self.group)
        r_scales = exchange(st["scales"], send_l, recv_l, self.group)
        r_eid = exchange(st["eid"], send_l, recv_l, self.group)
        f_recv = self.compute(r_codes, r_scales, r_eid)                   # (rows_recv, d) f32
        f_back = exchange(f_recv, recv_l, send_l, self.group)             # rows in send order
        return self.finish(st, f_back)

    __call__ = forward


class EPStep:
    """One rank's EP MoE step over fixed-capacity slots (csrc/ep.cu): no host
    synchronisation, fixed buffers, so the whole step — including the two
    equal-split all_to_alls — can be captured in a CUDA graph.

    Same arithmetic and the same combine order as EPMoE / the single-GPU layer
    (bitwise equal); slot padding costs exchange bytes, not compute (the
    expert kernels read the live row count from the device offsets).

    `layer` is this rank's MoELayer (expert_begin / n_local set), `n_tokens`
    the fixed batch per rank.  `all_to_all(out, inp)` defaults to
    dist.all_to_all_single over `group`."""

    def __init__(self, layer, n_tokens: int, rank: int, world: int, group=None, all_to_all=None):
        L = _lib.lib()
        self.layer, self.n, self.rank, self.world = layer, int(n_tokens), rank, world
        self.k, self.per, self.d = layer.top_k, layer.n_local, layer.d_model
        if layer.n_experts != self.per * world or layer.expert_begin != rank * self.per:
            raise ValueError("layer must hold experts [rank*per, (rank+1)*per) of n_experts = per*world")
        self.cap = self.n * min(self.k, self.per)
        self.slots = world * self.cap
        rb = L.cq_ep_row_bytes(self.d)
        dev = torch.device("cuda")
        self.send = torch.empty((self.slots, rb), dtype=torch.uint8, device=dev)
        self.recv = torch.empty_like(self.send)
        self.inv = torch.empty((self.n, self.k), dtype=torch.int32, device=dev)
        self.scratch = torch.empty(L.cq_ep_scratch_bytes(self.n, self.k, world, self.cap, self.per),
                                   dtype=torch.uint8, device=dev)
        self.codes_perm = torch.empty((self.slots, self.d), dtype=torch.int8, device=dev)
        self.scales_perm = torch.empty(self.slots, dtype=torch.float32, device=dev)
        self.offsets = torch.zeros(self.per + 1, dtype=torch.int32, device=dev)
        self.slot_of_row = torch.empty(self.slots, dtype=torch.int32, device=dev)
        self.fout = torch.empty((self.slots, self.d), dtype=torch.float32, device=dev)
        self.back = torch.empty_like(self.fout)
        self.ret = torch.empty_like(self.fout)
        self.out = torch.empty((self.n, self.d), dtype=torch.float32, device=dev)
        self.ws_route, _ = layer.workspace(self.n)
        self.tr = layer.trace(self.n)
        self.desc = layer.desc()
        offs = (ctypes.c_int64 * len(_lib.WS_NAMES))()   # expert-stage scratch, separate from routing's
        size = L.cq_moe_workspace(ctypes.byref(self.desc), -(-self.slots // self.k), offs)
        self.ws_exp = torch.empty(max(size, 256), dtype=torch.uint8, device=dev)
        if all_to_all is None:
            def all_to_all(out, inp):
                dist.all_to_all_single(out, inp, group=group)
        self.a2a = all_to_all

    def route_and_pack(self, x: torch.Tensor) -> None:
        L, tr = _lib.lib(), self.tr
        if x.shape != (self.n, self.d):
            raise ValueError(f"EPStep is built for ({self.n}, {self.d}) inputs, got {tuple(x.shape)}")
        _lib.check(L.cq_moe_route(ctypes.byref(self.desc), x.data_ptr(), _lib.dtype_code(x), self.n,
                                  self.ws_route.data_ptr(), self.ws_route.numel(), _lib.stream()))
        _lib.check(L.cq_ep_dispatch(tr["codes"].data_ptr(), tr["scales"].data_ptr(), tr["selected"].data_ptr(),
                                    self.n, self.k, self.d, self.per, self.world, self.cap, self.send.data_ptr(),
                                    self.inv.data_ptr(), self.scratch.data_ptr(), _lib.stream()))

    def run_experts(self) -> None:
        """recv -> grouped experts -> back (slot order)."""
        L = _lib.lib()
        _lib.check(L.cq_ep_group(self.recv.data_ptr(), self.slots, self.d, self.per, self.codes_perm.data_ptr(),
                                 self.scales_perm.data_ptr(), self.offsets.data_ptr(), self.slot_of_row.data_ptr(),
                                 self.scratch.data_ptr(), _lib.stream()))
        _lib.check(L.cq_moe_experts(ctypes.byref(self.desc), self.codes_perm.data_ptr(), self.scales_perm.data_ptr(),
                                    self.offsets.data_ptr(), self.slots, self.fout.data_ptr(),
                                    self.ws_exp.data_ptr(), self.ws_exp.numel(), _lib.stream()))
        _lib.check(L.cq_ep_scatter(self.fout.data_ptr(), self.offsets.data_ptr(), self.slot_of_row.data_ptr(),
                                   self.per, self.slots, self.d, self.back.data_ptr(), _lib.stream()))

    def combine(self, out: torch.Tensor | None = None) -> torch.Tensor:
        tr = self.tr
        out = self.out if out is None else out
        _lib.check(_lib.lib().cq_moe_combine(tr["selected"].data_ptr(), tr["weights"].data_ptr(),
                                             self.inv.data_ptr(), self.ret.data_ptr(), self.n, self.k, self.d,
                                             None, 0, out.data_ptr(), _lib.stream()))
        return out

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        self.route_and_pack(x)
        self.a2a(self.recv, self.send)
        self.run_experts()
        self.a2a(self.ret, self.back)
        return self.combine(out)


# ---------------------------------------------------------------------------
# Backends


class CudaBackend:
    """The B200 kernels.  `local` is a MoELayer built from this rank's experts
    with expert_begin/n_experts set (router weight replicated)."""

    def __init__(self, local):
        self.layer = local

    def route(self, x):
        lay = self.layer
        n = x.shape[0]
        buf, _ = lay.workspace(n)
        d = lay.desc()
        _lib.check(_lib.lib().cq_moe_route(ctypes.byref(d), x.data_ptr(), _lib.dtype_code(x), n, buf.data_ptr(),
                                           buf.numel(), _lib.stream()))
        tr = lay.trace(n)
        return tr["codes"], tr["scales"], tr["selected"], tr["weights"]

    def experts(self, codes, scales, eid, n_local):
        lay = self.layer
        rows = codes.shape[0]
        out = torch.zeros((rows, lay.d_model), dtype=torch.float32, device="cuda")
        offsets = torch.zeros(n_local + 1, dtype=torch.int32, device="cuda")
        if rows == 0:
            self.last = (codes, scales, offsets, 0)
            return out
        order = torch.sort(eid.long(), stable=True).indices
        counts = torch.bincount(eid.long(), minlength=n_local)
        offsets[1:] = torch.cumsum(counts, 0).to(torch.int32)
        g_codes, g_scales = codes[order].contiguous(), scales[order].contiguous()
        self.last = (g_codes, g_scales, offsets, rows)   # grouped inputs of the last call (profiling)
        f = torch.empty_like(out)
        # received row counts vary per step: size the workspace by the next power of two
        buf, _ = lay.workspace(1 << max(0, (-(-rows // lay.top_k) - 1).bit_length()))
        d = lay.desc()
        _lib.check(_lib.lib().cq_moe_experts(ctypes.byref(d), g_codes.data_ptr(), g_scales.data_ptr(),
                                             offsets.data_ptr(), rows, f.data_ptr(), buf.data_ptr(), buf.numel(),
                                             _lib.stream()))
        out[order] = f
        return out

    def combine(self, selected, weights, f_routes):
        n, k = selected.shape
        d = f_routes.shape[1]
        inv = torch.arange(n * k, dtype=torch.int32, device="cuda").view(n, k)
        out = torch.empty((n, d), dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().cq_moe_combine(selected.data_ptr(), weights.data_ptr(), inv.data_ptr(),
                                             f_routes.contiguous().data_ptr(), n, k, d, None, 0, out.data_ptr(),
                                             _lib.stream()))
        return out
