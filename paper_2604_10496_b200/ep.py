"""Expert parallelism for the MoE layer: experts sharded
over the ranks of one node, tokens data-parallel at the input, one exchange
each way.  The reference has no multi-GPU path: it evaluates every expert on
every token and masks (model.py:384-385, 391-401); this is the builder's
sharding of that block, with the same per-route arithmetic.

Per rank, one step:
  1. route its own tokens: A4 codes + scales, ordered router logits, top-k
     (bit-exact; `cq_moe_route`);
  2. dispatch: rows to the ranks that own the selected experts (experts
     [r*E/G, (r+1)*E/G) live on rank r).  A row carries the token's codes as
     packed nibbles (exact — quantization is per token and happens before
     routing, model.py:379), its scale and its routes to that rank;
  3. the owner groups the received routes by local expert and runs the
     grouped gate|up -> silu*up -> re-quantize -> down stage (`cq_moe_experts`);
  4. return: one fp32 row per received row;
  5. combine on the source rank, then + the replicated shared experts (DS;
     builder-defined, weight 1), which every rank runs on its
     own tokens while its dispatch is in flight.

Two row protocols (csrc/ep.cu header):
  * dedup=True: one row per (token, peer) however many of the token's experts
    the peer holds; the peer returns the weighted partial sum.  Exchange bytes
    scale with distinct peers per token, not with top_k.  Equal to the
    single-GPU layer up to the association of the fp32 adds across ranks
    (bitwise at world 1 and for tokens whose experts share a rank).
  * dedup=False: one row per route, outputs returned unweighted and combined
    on the source in ascending expert order: bitwise equal to the single-GPU
    layer for any world size.
Two sizings:
  * "fixed": every rank sends every peer `capacity` rows (the worst case);
    equal-split exchanges and no host read, so a whole step is one CUDA graph
    (decode);
  * "compact": per-peer row/route counts go first (one small all_to_all, one
    host read per step), then exact all_to_all-v splits (prefill).
`micro_batches` > 1 splits the rank's tokens so the exchange of batch m+1 and
the return of batch m-1 run on a communication stream while batch m's experts
run (routing is still one pass over all tokens).

`EPStep` is the device implementation (csrc/ep.cu + the layer kernels).  The
module-level protocol functions (`plan_rows`, `pack_rows`, `unpack_rows`) and
`EPMoE` restate the same protocol with torch index ops over a pluggable
compute backend; the world_size-2/4 gloo tests drive them on CPU with the
oracle as the backend, and the GPU tests check `EPStep`'s send rows against
`pack_rows` byte for byte.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib
from .errors import ConfigError, ShapeError


def expert_range(n_experts: int, world: int, rank: int) -> tuple[int, int]:
    if n_experts % world:
        raise ConfigError(f"{n_experts} experts do not split over {world} ranks")
    per = n_experts // world
    return rank * per, per


def routes_per_row(top_k: int, per: int, dedup: bool) -> int:
    return min(top_k, per) if dedup else 1


def header_bytes(kr: int) -> int:
    return (8 + 8 * kr + 15) // 16 * 16


def code_bytes(d: int) -> int:
    return d // 2 if d % 32 == 0 else d


# ---------------------------------------------------------------------------
# The row protocol restated with torch index ops (any device)


@dataclass
class RowPlan:
    tok: torch.Tensor       # (R,) token of each row, rows in send order (peer ascending, then token)
    dest: torch.Tensor      # (R,) peer
    m: torch.Tensor         # (R,) routes in the row
    e: torch.Tensor         # (R, kr) local expert ids ascending, -1 past m
    w: torch.Tensor         # (R, kr) receiver-side weights (1 in exact mode), 0 past m
    counts: torch.Tensor    # (G,) rows per peer
    routes: torch.Tensor    # (G,) routes per peer
    src_slot: torch.Tensor  # (n, k) row of the returned buffer per returned row of the token, -1 ends
    src_w: torch.Tensor     # (n, k) source-side weight of that row (1 in dedup mode)
    kr: int


def plan_rows(selected: torch.Tensor, weights: torch.Tensor, n_experts: int, world: int,
              dedup: bool = True) -> RowPlan:
    """Rows of one rank's dispatch (csrc/ep.cu ep_plan_kernel + ep_pack_kernel)."""
    n, k = selected.shape
    per = n_experts // world
    kr = routes_per_row(k, per, dedup)
    dev = selected.device
    e_sorted, idx = torch.sort(selected.long(), dim=1)               # ascending expert (ids distinct)
    w_sorted = torch.gather(weights.float(), 1, idx)
    dest = e_sorted // per
    new = torch.ones_like(dest, dtype=torch.bool)
    if dedup and k > 1:
        new[:, 1:] = dest[:, 1:] != dest[:, :-1]
    rid = (torch.cumsum(new.reshape(-1).long(), 0) - 1).view(n, k)    # row of each route (token order)
    pos = torch.arange(k, device=dev).expand(n, k)
    first = torch.cummax(torch.where(new, pos, torch.zeros_like(pos)), dim=1).values
    j = pos - first                                                   # route's place within its row
    R = int(new.sum())
    tok_r = torch.arange(n, device=dev)[:, None].expand(n, k)[new]
    dest_r = dest[new]
    e_r = torch.full((R, kr), -1, dtype=torch.int32, device=dev)
    w_r = torch.zeros((R, kr), dtype=torch.float32, device=dev)
    e_r[rid.reshape(-1), j.reshape(-1)] = (e_sorted - dest * per).reshape(-1).to(torch.int32)
    w_r[rid.reshape(-1), j.reshape(-1)] = (w_sorted if dedup else torch.ones_like(w_sorted)).reshape(-1)
    m_r = (e_r >= 0).sum(1).to(torch.int32)
    order = torch.sort(dest_r, stable=True).indices                   # send order: peer, then token
    slot = torch.empty(R, dtype=torch.long, device=dev)
    slot[order] = torch.arange(R, device=dev)
    row_in_tok = torch.cumsum(new.long(), 1) - 1
    src_slot = torch.full((n, k), -1, dtype=torch.int32, device=dev)
    src_w = torch.zeros((n, k), dtype=torch.float32, device=dev)
    ti, si = new.nonzero(as_tuple=True)
    src_slot[ti, row_in_tok[ti, si]] = slot[rid[ti, si]].to(torch.int32)
    src_w[ti, row_in_tok[ti, si]] = 1.0 if dedup else w_sorted[ti, si]
    counts = torch.bincount(dest_r, minlength=world).to(torch.int32)
    routes = torch.zeros(world, dtype=torch.int32, device=dev).index_add_(0, dest_r, m_r)
    return RowPlan(tok_r[order], dest_r[order], m_r[order], e_r[order], w_r[order], counts, routes, src_slot,
                   src_w, kr)


def pack_rows(codes: torch.Tensor, scales: torch.Tensor, plan: RowPlan) -> torch.Tensor:
    """(R, row_bytes) uint8 send rows, byte for byte what cq_ep_dispatch writes."""
    n, d = codes.shape
    c = codes[plan.tok]
    if d % 32 == 0:
        u = c.to(torch.uint8) & 0xF
        body = u[:, 0::2] | (u[:, 1::2] << 4)
    else:
        body = c.view(torch.uint8)
    R, kr = plan.e.shape
    h = torch.zeros((R, header_bytes(kr) // 4), dtype=torch.int32, device=codes.device)
    h[:, 0] = scales[plan.tok].float().view(torch.int32)
    h[:, 1] = plan.m
    h[:, 2:2 + 2 * kr:2] = plan.e
    h[:, 3:3 + 2 * kr:2] = plan.w.view(torch.int32)
    return torch.cat([body, h.view(torch.uint8)], dim=1)


def unpack_rows(rows: torch.Tensor, d: int, kr: int):
    """Received rows -> codes (R, d) int8, scales (R,), m (R,), e (R, kr), w (R, kr)."""
    cb = code_bytes(d)
    body, h = rows[:, :cb], rows[:, cb:].contiguous().view(torch.int32)
    if d % 32 == 0:
        lo, hi = body & 0xF, body >> 4
        nib = torch.stack([lo, hi], dim=2).reshape(rows.shape[0], d).to(torch.int16)
        codes = ((nib ^ 8) - 8).to(torch.int8)
    else:
        codes = body.contiguous().view(torch.int8)
    return (codes, h[:, 0].contiguous().view(torch.float32), h[:, 1], h[:, 2:2 + 2 * kr:2],
            h[:, 3:3 + 2 * kr:2].contiguous().view(torch.float32))


def _exchange(out, inp, out_splits, in_splits, group=None):
    dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits, group=group)


class EPMoE:
    """One rank of the EP layer in torch index ops over a compute backend
    (`route`, `experts`, `shared`): counts-first, compact exchanges, the same
    rows as EPStep.  Used by the CPU (gloo) tests of the protocol."""

    def __init__(self, backend, n_experts: int, top_k: int, rank: int, world: int, group=None, dedup: bool = True,
                 exchange=None):
        self.be, self.E, self.k, self.rank, self.world, self.group = backend, n_experts, top_k, rank, world, group
        self.begin, self.per = expert_range(n_experts, world, rank)
        self.dedup = dedup
        self.xchg = exchange or (lambda o, i, os_, is_: _exchange(o, i, os_, is_, group))
        self.last = {}

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        codes, scales, sel, wts = self.be.route(x)
        n, d = codes.shape
        plan = plan_rows(sel, wts, self.E, self.world, self.dedup)
        send = pack_rows(codes, scales, plan)
        cnt = torch.stack([plan.counts, plan.routes], 1).contiguous()   # (G, 2)
        rcnt = torch.empty_like(cnt)
        self.xchg(rcnt, cnt, None, None)
        s_split, r_split = plan.counts.tolist(), rcnt[:, 0].tolist()
        recv = torch.empty((sum(r_split), send.shape[1]), dtype=torch.uint8, device=send.device)
        self.xchg(recv, send, r_split, s_split)
        rc, rs, rm, re, rw = unpack_rows(recv, d, plan.kr)
        live = re >= 0
        ri, rj = live.nonzero(as_tuple=True)                             # routes in (row, j) order
        f = self.be.experts(rc[ri], rs[ri], re[ri, rj], self.per)         # (routes, d) f32
        back = torch.zeros((recv.shape[0], d), dtype=torch.float32, device=f.device)
        fj = torch.zeros((recv.shape[0], plan.kr, d), dtype=torch.float32, device=f.device)
        fj[ri, rj] = f
        if self.dedup:
            for j in range(plan.kr):                                    # ((0 + w0 f0) + w1 f1) ...
                on = rm > j
                back[on] = back[on] + rw[on, j, None] * fj[on, j]
        else:
            back = fj[:, 0].clone()
        ret = torch.empty((sum(s_split), d), dtype=torch.float32, device=f.device)
        self.xchg(ret, back, s_split, r_split)
        out = torch.zeros((n, d), dtype=torch.float32, device=f.device)
        for i in range(self.k):
            on = plan.src_slot[:, i] >= 0
            out[on] = out[on] + plan.src_w[on, i, None] * ret[plan.src_slot[on, i].long()]
        sh = self.be.shared(codes, scales) if hasattr(self.be, "shared") else None
        if sh is not None:
            for s in sh:
                out = out + s
        self.last = {"send_rows": send.shape[0], "recv_rows": recv.shape[0], "routes": int(ri.numel()),
                     "bytes_out": send.numel(), "bytes_back": back.numel() * 4}
        return out

    __call__ = forward


# ---------------------------------------------------------------------------
# Device implementation


class EPStep:
    """One rank's EP MoE step on the B200 kernels (csrc/ep.cu + the layer
    stages), fixed or compact sizing, dedup or exact rows, optional
    micro-batch overlap on a communication stream.

    `layer` is this rank's MoELayer (expert_begin / n_local set; shared experts
    replicated), `n_tokens` the batch per rank.  `exchange(out, inp,
    out_splits, in_splits)` defaults to dist.all_to_all_single over `group`
    (splits None = equal split)."""

    def __init__(self, layer, n_tokens: int, rank: int, world: int, group=None, *, dedup: bool = True,
                 sizing: str = "fixed", micro_batches: int = 1, exchange=None):
        L = _lib.lib()
        if sizing not in ("fixed", "compact"):
            raise ConfigError(f"sizing must be 'fixed' or 'compact', got {sizing!r}")
        self.layer, self.n, self.rank, self.world = layer, int(n_tokens), rank, world
        self.k, self.per, self.d = layer.top_k, layer.n_local, layer.d_model
        if layer.n_experts != self.per * world or layer.expert_begin != rank * self.per:
            raise ConfigError("layer must hold experts [rank*per, (rank+1)*per) of n_experts = per*world")
        if self.d % 16:
            raise ShapeError("expert parallelism needs d_model % 16 == 0")
        self.dedup, self.sizing = bool(dedup), sizing
        M = max(1, min(int(micro_batches), max(self.n, 1)))
        self.M = M
        self.bounds = [(m * self.n // M, (m + 1) * self.n // M) for m in range(M)]
        nmb = max(hi - lo for lo, hi in self.bounds)
        self.kr = routes_per_row(self.k, self.per, self.dedup)
        self.cap = nmb * (1 if self.dedup else min(self.k, self.per))  # rows per peer, worst case
        self.rows_max = world * self.cap
        self.rb = L.cq_ep_row_bytes(self.d, self.kr)
        dev = torch.device("cuda")
        z = dict(device=dev)
        self.send = [torch.zeros((self.rows_max, self.rb), dtype=torch.uint8, **z) for _ in range(M)]
        self.recv = [torch.zeros((self.rows_max, self.rb), dtype=torch.uint8, **z) for _ in range(M)]
        self.back = [torch.empty((self.rows_max, self.d), dtype=torch.float32, **z) for _ in range(M)]
        self.ret = [torch.empty((self.rows_max, self.d), dtype=torch.float32, **z) for _ in range(M)]
        self.src_slot = [torch.empty((hi - lo, self.k), dtype=torch.int32, **z) for lo, hi in self.bounds]
        self.src_w = [torch.empty((hi - lo, self.k), dtype=torch.float32, **z) for lo, hi in self.bounds]
        self.counts = torch.zeros((world, M, 2), dtype=torch.int32, **z)
        self.rcounts = torch.zeros_like(self.counts)
        routes_max = self.rows_max * self.kr
        self.codes_perm = torch.empty((routes_max, self.d), dtype=torch.int8, **z)
        self.scales_perm = torch.empty(routes_max, dtype=torch.float32, **z)
        self.offsets = torch.zeros(self.per + 1, dtype=torch.int32, **z)
        self.route_pos = torch.empty(routes_max, dtype=torch.int32, **z)
        self.fout = torch.empty((routes_max, self.d), dtype=torch.float32, **z)
        self.out = torch.empty((self.n, self.d), dtype=torch.float32, **z)
        self.scratch = torch.empty(L.cq_ep_scratch_bytes(nmb, self.k, self.rows_max, self.kr, self.per),
                                   dtype=torch.uint8, **z)
        self.ws_route, _ = layer.workspace(self.n)
        self.tr = layer.trace(self.n)
        self.desc = layer.desc()
        self.desc_route = layer.desc()
        self.desc_route.flags |= _lib.FLAG_SELECT_ONLY  # routing stops at the top-k: rows are planned here
        self.n_shared = layer.shared[0].n if layer.shared is not None else 0
        self.shared_out = (torch.empty((self.n_shared, self.n, self.d), dtype=torch.float32, **z)
                           if self.n_shared else None)
        offs = (ctypes.c_int64 * len(_lib.WS_NAMES))()   # expert-stage scratch, separate from routing's
        self.desc_exp = layer.desc()  # expert stage over received rows: shared experts run separately
        self.desc_exp.flags &= ~_lib.FLAG_SHARED_MERGED
        size = L.cq_moe_workspace(ctypes.byref(self.desc_exp), -(-routes_max // self.k), offs)
        self.ws_exp = torch.empty(max(size, 256), dtype=torch.uint8, **z)
        self.xchg = exchange or (lambda o, i, os_, is_: _exchange(o, i, os_, is_, group))
        self.comm = torch.cuda.Stream()
        mk = lambda: [torch.cuda.Event() for _ in range(M)]  # noqa: E731
        self.ev_packed, self.ev_recv, self.ev_back, self.ev_ret = torch.cuda.Event(), mk(), mk(), mk()
        self._host_counts = None

    # ---- phases (the in-process multi-rank tests drive these directly) ----
    def dispatch(self, x: torch.Tensor) -> None:
        """Route all tokens, then pack every micro-batch's send rows."""
        L, tr = _lib.lib(), self.tr
        if x.shape != (self.n, self.d):
            raise ShapeError(f"EPStep is built for ({self.n}, {self.d}) inputs, got {tuple(x.shape)}")
        _lib.check(L.cq_moe_route(ctypes.byref(self.desc_route), x.data_ptr(), _lib.dtype_code(x), self.n,
                                  self.ws_route.data_ptr(), self.ws_route.numel(), _lib.stream()))
        cap = self.cap if self.sizing == "fixed" else 0
        for m, (lo, hi) in enumerate(self.bounds):
            _lib.check(L.cq_ep_dispatch(
                tr["codes"][lo:].data_ptr(), tr["scales"][lo:].data_ptr(), tr["selected"][lo:].data_ptr(),
                tr["weights"][lo:].data_ptr(), hi - lo, self.k, self.d, self.per, self.world, int(self.dedup), cap,
                self.send[m].data_ptr(), self.counts[:, m].data_ptr(), 2 * self.M, self.src_slot[m].data_ptr(),
                self.src_w[m].data_ptr(), self.scratch.data_ptr(), _lib.stream()))

    def run_shared(self) -> None:
        if self.n_shared:
            _lib.check(_lib.lib().cq_moe_shared_experts(ctypes.byref(self.desc), self.n, self.shared_out.data_ptr(),
                                                        self.ws_route.data_ptr(), self.ws_route.numel(),
                                                        _lib.stream()))

    def read_counts(self) -> None:
        """Compact sizing: one host read of the sent and received counts."""
        self._host_counts = (self.counts.cpu(), self.rcounts.cpu())

    def splits(self, m: int):
        """(send_splits, recv_splits) in rows for micro-batch m (None: equal split of cap rows)."""
        if self.sizing == "fixed":
            return None, None
        sc, rc = self._host_counts
        return sc[:, m, 0].tolist(), rc[:, m, 0].tolist()

    def views(self, m: int):
        """(send, recv, back, ret) views holding micro-batch m's live rows."""
        s, r = self.splits(m)
        if s is None:
            return self.send[m], self.recv[m], self.back[m], self.ret[m]
        ns, nr = sum(s), sum(r)
        return self.send[m][:ns], self.recv[m][:nr], self.back[m][:nr], self.ret[m][:ns]

    def experts(self, m: int) -> None:
        """recv[m] -> grouped experts -> back[m] (one row per received row)."""
        L = _lib.lib()
        if self.sizing == "fixed":
            rows, routes = self.rows_max, self.rows_max * self.kr
        else:
            rows, routes = sum(self.splits(m)[1]), int(self._host_counts[1][:, m, 1].sum())
        _lib.check(L.cq_ep_group(self.recv[m].data_ptr(), rows, self.d, self.kr, self.per, self.codes_perm.data_ptr(),
                                 self.scales_perm.data_ptr(), self.offsets.data_ptr(), self.route_pos.data_ptr(),
                                 self.scratch.data_ptr(), _lib.stream()))
        if routes:
            _lib.check(L.cq_moe_experts(ctypes.byref(self.desc_exp), self.codes_perm.data_ptr(),
                                        self.scales_perm.data_ptr(), self.offsets.data_ptr(), routes,
                                        self.fout.data_ptr(), self.ws_exp.data_ptr(), self.ws_exp.numel(),
                                        _lib.stream()))
        _lib.check(L.cq_ep_partial(self.fout.data_ptr(), self.route_pos.data_ptr(), self.recv[m].data_ptr(), rows,
                                   self.d, self.kr, int(not self.dedup), self.back[m].data_ptr(), _lib.stream()))

    def combine(self, m: int, out: torch.Tensor) -> None:
        lo, hi = self.bounds[m]
        add = self.shared_out[:, lo:].data_ptr() if self.n_shared else None
        _lib.check(_lib.lib().cq_ep_combine(self.ret[m].data_ptr(), self.src_slot[m].data_ptr(),
                                            self.src_w[m].data_ptr(), hi - lo, self.k, self.d, add, self.n_shared,
                                            self.n * self.d, out[lo:].data_ptr(), _lib.stream()))

    def exchange_bytes(self) -> dict:
        """Bytes this rank sent in the last step (compact: live rows; fixed: the slots)."""
        if self.sizing == "fixed":
            return {"out": self.M * self.rows_max * self.rb, "back": self.M * self.rows_max * self.d * 4}
        sc, rc = self._host_counts
        return {"out": int(sc[:, :, 0].sum()) * self.rb, "back": int(rc[:, :, 0].sum()) * self.d * 4}

    # ---- the whole step ----
    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        out = self.out if out is None else out
        cs, comm = torch.cuda.current_stream(), self.comm
        self.dispatch(x)
        if self.sizing == "compact":
            self.xchg(self.rcounts, self.counts, None, None)
            self.read_counts()
        self.ev_packed.record(cs)
        self.run_shared()                      # overlaps the first dispatch exchange
        comm.wait_event(self.ev_packed)

        def out_xchg(m):
            s, r = self.splits(m)
            snd, rcv, _, _ = self.views(m)
            with torch.cuda.stream(comm):
                self.xchg(rcv, snd, r, s)
                self.ev_recv[m].record(comm)

        out_xchg(0)
        for m in range(self.M):
            if m + 1 < self.M:
                out_xchg(m + 1)                # issued before the return of m: it never waits on m's experts
            cs.wait_event(self.ev_recv[m])
            self.experts(m)
            self.ev_back[m].record(cs)
            s, r = self.splits(m)
            _, _, bck, rt = self.views(m)
            with torch.cuda.stream(comm):
                comm.wait_event(self.ev_back[m])
                self.xchg(rt, bck, s, r)
                self.ev_ret[m].record(comm)
        for m in range(self.M):
            cs.wait_event(self.ev_ret[m])
            self.combine(m, out)
        return out
