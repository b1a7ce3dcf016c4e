"""Attention-site LUT GEMMs: the q / k / v / out
projections of a decoder layer on the same tcgen05 LUT kernel as the experts.

Reference semantics (model.py:353-375): q, k and v read one fake-quantized
copy of the normed input (the `_site_value` cache, model.py:312-321), so here
the three codebooks are stacked along d_out and run as ONE launch on one A4
quantization; `out` quantizes the attention output separately.  Dense shapes,
no routing.  A row's result depends only on its own codebook row and the
codes, so the stacked launch is bitwise equal to three separate ones.
"""

from __future__ import annotations

import torch

from .errors import ShapeError
from .lutgemm import PackedClusteredWeights, lut_gemm_tc
from .quant import QuantSpec, quantize_activations


def stack_rows(pws) -> PackedClusteredWeights:
    """Codebooks of equal (d_in, group_size) laid end to end along d_out."""
    pws = list(pws)
    d_in, g = pws[0].d_in, pws[0].group_size
    for pw in pws:
        if (pw.d_in, pw.group_size) != (d_in, g):
            raise ShapeError("stacked sites must share d_in and group_size")
    cents = torch.cat([pw.centroids for pw in pws]).contiguous()
    ids = torch.cat([pw.ids_packed for pw in pws]).contiguous()
    return PackedClusteredWeights(cents, ids, d_in, g)


class QKVLinear:
    """q, k, v = x @ W_q, x @ W_k, x @ W_v on one shared A4 quantization of x."""

    def __init__(self, q: PackedClusteredWeights, k: PackedClusteredWeights, v: PackedClusteredWeights,
                 planes: int = 3, layout: str = "umma128u"):
        self.widths = (q.d_out, k.d_out, v.d_out)
        self.d_in = q.d_in
        self.w = stack_rows((q, k, v))
        self.planes, self.layout = planes, layout
        self.w.prepare_tc(planes, layout)

    def __call__(self, x, spec: QuantSpec = QuantSpec(4)):
        """x: (N, d_in) -> (q, k, v) float32 views of one (N, sum d_out) result."""
        qa = quantize_activations(x, spec, check_finite=False)
        out = lut_gemm_tc(qa, self.w, self.planes, self.layout)
        return tuple(torch.split(out, self.widths, dim=1))


class OutLinear:
    """attn_proj = A4(attn_out) @ W_out (model.py:370-372)."""

    def __init__(self, w: PackedClusteredWeights, planes: int = 3, layout: str = "umma128u"):
        self.w, self.planes, self.layout = w, planes, layout
        self.w.prepare_tc(planes, layout)

    def __call__(self, x, spec: QuantSpec = QuantSpec(4)) -> torch.Tensor:
        return lut_gemm_tc(quantize_activations(x, spec, check_finite=False), self.w, self.planes, self.layout)
