"""Generate tests/golden/tiny_model.cqm1 with the REFERENCE's own container
writer (container.py save_model), plus tiny_model_ref.npz: what the
reference's read_container / load_model returns for the expert codebooks and
router weights, and the composed-oracle MoE outputs for a fixed input.

Run in the build container (needs /root/reference); the outputs are committed.

    python tests/golden/make_cqm1.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from codequant.container import load_model, read_container, save_model  # noqa: E402
from codequant.model import (DecoderLayerWeights, ModelConfig, ModelWeights,  # noqa: E402
                             codebook_to_dense, site_path)

from oracle import oracle as o  # noqa: E402


def main():
    rng = np.random.default_rng(2604)
    d, ff, E, k, L = 128, 128, 4, 2, 2
    cfg = ModelConfig(d_model=d, n_heads=2, d_ff=ff, n_experts=E, top_k=k, n_layers=L, n_calib=1, seed=7)
    codebooks, layers = {}, []
    # layer 0: g = 128 (tensor-core envelope); layer 1: g = 32 and one K = 8 codebook (padding)
    for li, g in ((0, 128), (1, 32)):
        def clustered(name, d_in, d_out, kc=16):
            cents = (rng.standard_normal((d_out, d_in // g, kc)) / np.sqrt(d_in)).astype(np.float32)
            ids = rng.integers(0, kc, (d_out, d_in)).astype(np.uint8)
            codebooks[name] = (cents, ids, g)
            return codebook_to_dense(cents.astype(np.float64), ids, g)

        def dense(*shape):
            return rng.standard_normal(shape) / np.sqrt(shape[0])

        gate, up, down = [], [], []
        for e in range(E):
            gate.append(clustered(site_path(li, "gate", e), d, ff, 8 if (li, e) == (1, 0) else 16))
            up.append(clustered(site_path(li, "up", e), d, ff))
            down.append(clustered(site_path(li, "down", e), ff, d))
        layers.append(DecoderLayerWeights(a1=np.ones(d), a2=np.ones(d), w_q=dense(d, d), w_k=dense(d, d),
                                          w_v=dense(d, d), w_out=dense(d, d),
                                          w_router=dense(d, E).astype(np.float32).astype(np.float64),
                                          w_gate=gate, w_up=up, w_down=down))
    w = ModelWeights(cfg, layers, {"origin": "make_cqm1"}, codebooks)
    path = os.path.join(HERE, "tiny_model.cqm1")
    save_model(w, path)

    # what the reference reads back
    config, tensors = read_container(path)
    back = load_model(path, dtype=np.float32)
    ref = {}
    x = rng.standard_normal((24, d)).astype(np.float32)
    ref["x"] = x
    for li in range(L):
        ref[f"router{li}"] = tensors[site_path(li, "router")][1]
        experts = []
        for e in range(E):
            mats = []
            for s in ("gate", "up", "down"):
                cents, ids, g = back.codebooks[site_path(li, s, e)]
                ref[f"l{li}e{e}{s}_centroids"] = np.asarray(cents, np.float32)
                ref[f"l{li}e{e}{s}_ids"] = np.asarray(ids, np.uint8)
                ref[f"l{li}e{e}{s}_g"] = np.int64(g)
                c16 = np.zeros(cents.shape[:2] + (16,), np.float32)
                c16[:, :, :cents.shape[2]] = cents
                mats.append((c16, o.pack_ids(np.asarray(ids, np.uint8)), g))
            experts.append(mats)
        ref[f"out{li}"] = o.moe_layer(x, np.asarray(ref[f"router{li}"], np.float32), experts, k)
    ref["config"] = np.array([f"{kk}={vv}" for kk, vv in sorted(config.items())])
    np.savez_compressed(os.path.join(HERE, "tiny_model_ref.npz"), **ref)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
