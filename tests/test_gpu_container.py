"""CQM1 container -> device MoE layers: the layers built from a container the
reference wrote reproduce the composed reference path on the same codebooks
(layer 0: g = 128, tensor-core path; layer 1: g = 32 with a K = 8 codebook,
fp32 path)."""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import oracle as o  # noqa: E402
from paper_2604_10496_b200.container import moe_layers_from_container  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def test_container_layers_match_reference_composition():
    ref = np.load(os.path.join(HERE, "golden", "tiny_model_ref.npz"))
    layers = moe_layers_from_container(os.path.join(HERE, "golden", "tiny_model.cqm1"))
    x = torch.from_numpy(ref["x"]).cuda()
    assert layers[0].gate.tc is not None and layers[1].gate.tc is None
    for li, layer in enumerate(layers):
        out = layer(x).cpu().numpy()
        assert o.relative_error(out, ref[f"out{li}"]) <= (1e-3 if li == 0 else 1e-5)
        ordered = layer(x, path="ordered").cpu().numpy()
        assert np.array_equal(ordered.view(np.int32), ref[f"out{li}"].view(np.int32)) or \
            o.relative_error(ordered, ref[f"out{li}"]) <= 1e-6
