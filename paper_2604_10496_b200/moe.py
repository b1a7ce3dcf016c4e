"""MoE-layer operator: the MoE block of the reference's forward pass
(model.py:377-404) as one device call (`cq_moe_forward`).

Inputs are the reference's own formats, unchanged: a full-precision router
weight (d_model, E) (pipeline.py:455-467), per-expert PackedClusteredWeights
for gate / up / down (lutgemm.py:53-87) and an optional rotation matrix R
(rotation.py:83-87; applied online as v = x @ R, pipeline.py:516).  The
weights are stacked per site once at construction so one grouped launch
covers every expert.

Semantics (bit-exact where the reference is integer/ordered):
codes = A4(v); logits = ordered (codes*s) @ W_router; top-k stable, softmax
over the selected; per expert e ascending over its routed tokens
h = silu(gate) * up, d = down(A4(h)); out = sum_e w_e * d_e (e ascending).
Builder-defined (not in the reference): token permutation into expert
segments; shared experts added with weight 1 after the routed sum.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, DivergenceError, ShapeError
from .lutgemm import PackedClusteredWeights, prepare_tc_site

_PATHS = {"auto": _lib.CQ_PATH_AUTO, "f32": _lib.CQ_PATH_F32, "tc": _lib.CQ_PATH_TC,
          "ordered": _lib.CQ_PATH_ORDERED}


@dataclass
class ExpertStack:
    """One site (gate, up or down) of several experts laid end to end."""

    ids: torch.Tensor        # (E, d_out, d_in/2) uint8
    centroids: torch.Tensor  # (E, d_out, d_in/g, 16) float32
    d_in: int
    d_out: int
    group_size: int          # 0: embedding-wise (one group per row, g = d_in)
    tc: dict | None = None

    def __post_init__(self):
        if self.group_size == 0:
            self.group_size = self.d_in

    @classmethod
    def from_packed(cls, pws) -> "ExpertStack":
        pws = list(pws)
        if not pws:
            raise ShapeError("no experts")
        d_in, d_out, g = pws[0].d_in, pws[0].d_out, pws[0].group_size
        for pw in pws:
            if (pw.d_in, pw.d_out, pw.group_size) != (d_in, d_out, g):
                raise ShapeError("experts of one site must share (d_in, d_out, group_size)")
        if d_in % 2:
            raise ShapeError("stacked expert sites need an even input dimension")
        ids = torch.stack([pw.ids_packed for pw in pws]).contiguous()
        cents = torch.stack([pw.centroids for pw in pws]).contiguous()
        return cls(ids, cents, d_in, d_out, g)

    @property
    def n(self) -> int:
        return self.ids.shape[0]

    def prepare_tc(self, planes: int, layout: str = "umma128u", out=None) -> None:
        """out: (ids, lut, rowscale) destination views (a merged routed + shared buffer)."""
        if out is not None or self.tc is None or (self.tc["planes"], self.tc["layout"]) != (planes, layout):
            rows = self.n * self.d_out
            self.tc = prepare_tc_site(self.ids.view(rows, -1), self.centroids.view(rows, -1, 16),
                                      rows, self.d_in, self.group_size, planes, layout, out=out)

    def site(self, tc: dict | None = None) -> _lib.ExpertSite:
        """tc: tensor-core data to describe instead of self.tc (a layer's merged copy)."""
        s = _lib.ExpertSite()
        s.ids = self.ids.data_ptr()
        s.centroids = self.centroids.data_ptr()
        s.group_size = self.group_size
        tc = tc if tc is not None else self.tc
        if tc is not None:
            s.tc_ids = tc["ids"].data_ptr()
            s.tc_lut = tc["lut"].data_ptr()
            s.tc_rowscale = tc["rowscale"].data_ptr()
            s.tc_planes = tc["planes"]
            s.tc_layout = _lib.TC_LAYOUTS[tc["kernel_layout"]]
        return s


def _as_f32_device(a) -> torch.Tensor:
    if not isinstance(a, torch.Tensor):
        a = torch.from_numpy(np.ascontiguousarray(np.asarray(a), dtype=np.float32))
    return a.to(device="cuda", dtype=torch.float32).contiguous()


class MoELayer:
    """A routed MoE FFN block on prepared device weights.

    experts: sequence of (gate, up, down) PackedClusteredWeights, one per expert
    (or pre-stacked ExpertStack triples via `from_stacks`).  `path`: "auto"
    (tensor-core path when prepared, else fp32 LUT-GEMV), "f32", "tc",
    "ordered" (bit-exact chains, the GPU-side oracle).
    """

    def __init__(self, w_router, experts, top_k: int, rotation=None, shared=(), path: str = "auto",
                 expert_begin: int = 0, n_experts: int | None = None):
        stacks = list(zip(*experts)) if experts else ([], [], [])
        self.gate = ExpertStack.from_packed(stacks[0])
        self.up = ExpertStack.from_packed(stacks[1])
        self.down = ExpertStack.from_packed(stacks[2])
        self._init(w_router, top_k, rotation, shared, path, expert_begin, n_experts)

    @classmethod
    def from_stacks(cls, w_router, gate: ExpertStack, up: ExpertStack, down: ExpertStack, top_k: int,
                    rotation=None, shared=None, path: str = "auto", expert_begin: int = 0,
                    n_experts: int | None = None) -> "MoELayer":
        self = cls.__new__(cls)
        self.gate, self.up, self.down = gate, up, down
        self._init(w_router, top_k, rotation, shared or (), path, expert_begin, n_experts)
        return self

    def _init(self, w_router, top_k, rotation, shared, path, expert_begin, n_experts):
        self.w_router = _as_f32_device(w_router)
        self.d_model = self.gate.d_in
        self.d_ff = self.gate.d_out
        self.n_local = self.gate.n
        self.n_experts = n_experts if n_experts is not None else self.n_local
        self.expert_begin = expert_begin
        if self.w_router.shape != (self.d_model, self.n_experts):
            raise ShapeError(f"router weight {tuple(self.w_router.shape)} != "
                             f"({self.d_model}, {self.n_experts})")
        if self.up.d_in != self.d_model or self.up.d_out != self.d_ff:
            raise ShapeError("up projection shape does not match gate")
        if self.down.d_in != self.d_ff or self.down.d_out != self.d_model:
            raise ShapeError("down projection shape does not match (d_ff, d_model)")
        if not 1 <= top_k <= min(16, self.n_experts):
            raise ConfigError(f"top_k {top_k} outside [1, min(16, n_experts)]")
        self.top_k = int(top_k)
        self.rotation = None if rotation is None else _as_f32_device(rotation)
        if self.rotation is not None and self.rotation.shape != (self.d_model, self.d_model):
            raise ShapeError("rotation must be (d_model, d_model)")
        if isinstance(shared, tuple) and len(shared) == 3 and isinstance(shared[0], ExpertStack):
            self.shared = shared
        elif shared:
            sh = list(zip(*shared))
            self.shared = tuple(ExpertStack.from_packed(s) for s in sh)
        else:
            self.shared = None
        if path not in _PATHS:
            raise ConfigError(f"unknown path {path!r}; one of {sorted(_PATHS)}")
        self.path = path
        # store h = silu(a) * b in the workspace on the tensor-core path too (trace(); costs an
        # fp32 write of every routed hidden row)
        self.keep_hidden = False
        # tensor-core path with the ordered (bit-exact) rotation instead of the tcgen05 one:
        # routing then matches the reference bit for bit, at CUDA-core speed
        self.exact_rotation = False
        self._ws = {}
        self._rot_tc = None  # R as three bf16 planes for the tensor-core rotation (prepare_tc)
        self._sh_tc = None  # this layer's tensor-core copy of the shared experts (merged with the routed)

    # ------------------------------------------------------------------
    def tc_shapes_ok(self) -> bool:
        """The tcgen05 path's envelope: 128 | d_model, d_ff, and every group size."""
        sites = [self.gate, self.up, self.down] + (list(self.shared) if self.shared is not None else [])
        return all(s.d_in % 128 == 0 and s.d_out % 128 == 0 and s.group_size % 128 == 0 for s in sites)

    def prepare_tc(self, planes_gate_up: int = 3, planes_down: int = 2,
                   layout: str = "umma128u") -> "MoELayer":
        """tcgen05 layouts (unsigned base-128 digit planes): 3 planes where the
        output is re-quantized (gate, up), 2 for down."""
        sites = [(self.gate, planes_gate_up), (self.up, planes_gate_up), (self.down, planes_down)]
        if self._can_merge_shared():
            # routed and shared experts of a site in one buffer (shared after the routed ones), so the
            # forward runs the shared experts as extra segments of the routed grouped launches
            # routed and shared experts of a site in one buffer (shared after the routed ones), so the
            # forward runs the shared experts as extra segments of the routed grouped launches.  The
            # shared stacks may be shared by several layers (EP shards): their copy is this layer's
            # (self._sh_tc), never written into the stack
            self._sh_tc = []
            for (r, p), sh in zip(sites, self.shared):
                rows_r, rows_s = r.n * r.d_out, sh.n * sh.d_out
                ids = torch.empty((rows_r + rows_s, r.d_in // 2), dtype=torch.uint8, device="cuda")
                lut = torch.empty((rows_r + rows_s, r.d_in // r.group_size, p, 16), dtype=torch.int8, device="cuda")
                rs = torch.empty((rows_r + rows_s,), dtype=torch.float32, device="cuda")
                r.prepare_tc(p, layout, out=(ids[:rows_r], lut[:rows_r], rs[:rows_r]))
                tail = prepare_tc_site(sh.ids.view(rows_s, -1), sh.centroids.view(rows_s, -1, 16), rows_s, sh.d_in,
                                       sh.group_size, p, layout, out=(ids[rows_r:], lut[rows_r:], rs[rows_r:]))
                if r.tc["kernel_layout"] != tail["kernel_layout"]:  # one launch, one lookup kernel
                    r.tc["kernel_layout"] = tail["kernel_layout"] = layout
                self._sh_tc.append(tail)
        else:
            self._sh_tc = None
            if self.shared is not None:
                sites += [(self.shared[0], planes_gate_up), (self.shared[1], planes_gate_up),
                          (self.shared[2], planes_down)]
            for s, p in sites:
                s.prepare_tc(p, layout)
        if self.rotation is not None and self.d_model % 256 == 0 and self._rot_tc is None:
            lib = _lib.lib()
            buf = torch.empty(lib.cq_rotation_prepared_bytes(self.d_model), dtype=torch.uint8, device="cuda")
            _lib.check(lib.cq_rotation_prepare(self.rotation.data_ptr(), self.d_model, buf.data_ptr(),
                                               _lib.stream()))
            self._rot_tc = buf
            self._ws = {}
        return self

    def _can_merge_shared(self) -> bool:
        if self.shared is None:
            return False
        return all((sh.d_in, sh.d_out, sh.group_size) == (r.d_in, r.d_out, r.group_size)
                   for r, sh in zip((self.gate, self.up, self.down), self.shared))

    def shared_merged(self) -> bool:
        """The shared experts' tensor-core data directly follows the routed experts' in every site
        (prepare_tc of this layer), so cq_moe_forward may run them as extra segments."""
        if not self._can_merge_shared():
            return False
        if self._sh_tc is None:
            return False
        for r, tail in zip((self.gate, self.up, self.down), self._sh_tc):
            if r.tc is None:
                return False
            for key in ("ids", "lut", "rowscale"):
                a, b = r.tc[key], tail[key]
                if a.data_ptr() + a.numel() * a.element_size() != b.data_ptr():
                    return False
            if r.tc["kernel_layout"] != tail["kernel_layout"] or r.tc["planes"] != tail["planes"]:
                return False
        return True

    def desc(self, path: str | None = None) -> _lib.MoEDesc:
        d = _lib.MoEDesc()
        d.d_model, d.d_ff, d.n_experts, d.top_k = self.d_model, self.d_ff, self.n_experts, self.top_k
        d.n_local_experts, d.expert_begin = self.n_local, self.expert_begin
        d.w_router = self.w_router.data_ptr()
        d.rotation = self.rotation.data_ptr() if self.rotation is not None else None
        d.gate, d.up, d.down = self.gate.site(), self.up.site(), self.down.site()
        if self.shared is not None:
            d.n_shared = self.shared[0].n
            sh_tc = self._sh_tc or (None, None, None)
            d.sh_gate, d.sh_up, d.sh_down = (s.site(t) for s, t in zip(self.shared, sh_tc))
        d.path = _PATHS[path or self.path]
        d.flags = _lib.FLAG_KEEP_HIDDEN if self.keep_hidden else 0
        # CQ_SHARED_MERGE=0: separate shared-expert launches (A/B measurement)
        if ((path or self.path) in ("tc", "auto") and os.environ.get("CQ_SHARED_MERGE", "1") != "0"
                and self.shared_merged()):
            d.flags |= _lib.FLAG_SHARED_MERGED
        # the tensor-core rotation goes with the tensor-core path; f32 / ordered keep the fp32 rotation
        if self._rot_tc is not None and (path or self.path) in ("tc", "auto") and not self.exact_rotation:
            d.rotation_tc = self._rot_tc.data_ptr()
        return d

    def workspace(self, n: int, path: str | None = None):
        d = self.desc(path)
        key = (n, path or self.path, self.exact_rotation, d.flags)  # the layout follows the flags
        if key not in self._ws:
            offs = (ctypes.c_int64 * len(_lib.WS_NAMES))()
            size = _lib.load_library().cq_moe_workspace(ctypes.byref(d), n, offs)
            buf = torch.empty(max(size, 256), dtype=torch.uint8, device="cuda")
            o = offs[_lib.WS_NAMES.index("status")]
            buf[o:o + 16].zero_()  # sticky non-finite flags: cleared here, only ever set by the layer
            self._ws[key] = (buf, list(offs))
        return self._ws[key]

    def check_finite(self, n: int, path: str | None = None) -> None:
        """Read (one host sync) and clear the non-finite flags the last forwards
        over n tokens set; raise DivergenceError naming the site like the
        reference (model.py:307-309, quant.py:93-94)."""
        buf, offs = self.workspace(n, path)
        o = offs[_lib.WS_NAMES.index("status")]
        st = buf[o:o + 16].view(torch.int32)
        flags = st.tolist()
        if flags[0] or flags[1]:
            st.zero_()
            site = "router/gate/up input" if flags[0] else "down input (silu(gate) * up)"
            raise DivergenceError(f"non-finite values at MoE site {site!r}")

    def forward(self, x, out: torch.Tensor | None = None, path: str | None = None,
                check_finite: bool = False) -> torch.Tensor:
        """x: (N, d_model) float32/bfloat16 CUDA tensor -> moe_sum (N, d_model) float32.

        No host synchronisation unless `check_finite` (then DivergenceError on
        non-finite input or hidden, like the reference); otherwise the flags
        stay set for a later `check_finite(n)`."""
        if not isinstance(x, torch.Tensor):
            x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
        x = x.to("cuda").contiguous()
        if x.dim() != 2 or x.shape[1] != self.d_model:
            raise ShapeError(f"input has shape {tuple(x.shape)}, layer expects (N, {self.d_model})")
        if self.n_local != self.n_experts or self.expert_begin != 0:
            raise ConfigError("sharded layer: use paper_2604_10496_b200.ep.EPMoE")
        n = x.shape[0]
        if out is None:
            out = torch.empty((n, self.d_model), dtype=torch.float32, device="cuda")
        buf, _ = self.workspace(n, path)
        d = self.desc(path)
        _lib.check(_lib.lib().cq_moe_forward(ctypes.byref(d), x.data_ptr(), _lib.dtype_code(x), n,
                                             out.data_ptr(), buf.data_ptr(), buf.numel(), _lib.stream()))
        if check_finite:
            self.check_finite(n, path)
        return out

    __call__ = forward

    def route(self, x, path: str | None = None) -> None:
        """The routing stage alone (`cq_moe_route`) into the workspace: codes,
        logits, top-k, the segment permutation and the gathered codes_perm /
        scales_perm.  (The tensor-core forward gathers inside its GEMM's B build
        and leaves codes_perm unwritten.)"""
        x = x.to("cuda").contiguous()
        n = x.shape[0]
        buf, _ = self.workspace(n, path)
        d = self.desc(path)
        _lib.check(_lib.lib().cq_moe_route(ctypes.byref(d), x.data_ptr(), _lib.dtype_code(x), n, buf.data_ptr(),
                                           buf.numel(), _lib.stream()))

    def trace(self, n: int, path: str | None = None) -> dict:
        """Views of the workspace buffers of the last forward over n tokens.
        "hidden" is h = silu(a) * b on the tensor-core path only with
        `keep_hidden` set before that forward (else the gate output), and
        "hcodes" (row-major) likewise: without it the re-quantizer writes the
        codes only into the down GEMM's operand tiles."""
        buf, offs = self.workspace(n, path)
        k, d, ff, E, R = self.top_k, self.d_model, self.d_ff, self.n_experts, n * self.top_k
        spec = {"codes": (torch.int8, (n, d)), "scales": (torch.float32, (n,)),
                "logits": (torch.float32, (n, E)), "selected": (torch.int32, (n, k)),
                "weights": (torch.float32, (n, k)), "counts": (torch.int32, (E + 1,)),
                "offsets": (torch.int32, (self.n_local + 1,)),
                "perm_token": (torch.int32, (R,)), "perm_slot": (torch.int32, (R,)),
                "inv": (torch.int32, (n, k)), "codes_perm": (torch.int8, (R, d)),
                "scales_perm": (torch.float32, (R,)), "hidden": (torch.float32, (R, ff)),
                "hcodes": (torch.int8, (R, ff)), "hscales": (torch.float32, (R,)),
                "fout": (torch.float32, (R, d)), "tok_sums": (torch.int32, (n,)),
                "status": (torch.int32, (4,))}
        res = {}
        for name, (dt, shape) in spec.items():
            o = offs[_lib.WS_NAMES.index(name)]
            numel = int(np.prod(shape))
            res[name] = buf[o:o + numel * torch.tensor([], dtype=dt).element_size()].view(dt).view(shape)
        return res


def moe_layer(v, w_router, experts, top_k: int, rotation=None, shared=(), path: str = "auto"):
    """One-shot functional form: build the layer (tcgen05 layouts prepared when
    the shapes allow and the path is "auto" / "tc") and run it on v, raising
    DivergenceError on non-finite values like the reference's forward."""
    layer = MoELayer(w_router, experts, top_k, rotation=rotation, shared=shared, path=path)
    if path in ("auto", "tc") and layer.tc_shapes_ok():
        layer.prepare_tc()
    return layer.forward(v, check_finite=True)
