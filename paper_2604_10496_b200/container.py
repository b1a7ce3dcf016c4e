"""CQM1 model container -> device MoE layers.

Restates the reader of the reference's single-file container
(`container.py:1-13` layout, `:103-165` read_container) and builds one
`MoELayer` per decoder layer from the clustered expert sites, so calibrated
codebooks (fp32 centroids that are not bf16-exact) feed the B200 kernels
directly.

Layout (little-endian): magic "CQM1" | u32 version = 1 | u64 text_len |
config text ("key = value" lines) | u32 n_tensors | per tensor: u32 name_len |
name | u8 dtype | u32 ndim | u64 dims... | payload.  dtype 0 = float32,
1 = 4-bit ids packed low nibble first across the flattened array, 2 = int8.
A clustered site stores "<site>.centroids" (d_out, n_groups, K) f32 and
"<site>.ids" (d_out, d_in) nibbles instead of its dense weight
(`container.py:194-201`).

Ids are re-packed per row (what PackedClusteredWeights expects,
lutgemm.py:111-116); for even d_in the bytes are the container's own.
"""

from __future__ import annotations

import struct

import numpy as np

from .errors import ConfigError, FormatError

MAGIC = b"CQM1"
VERSION = 1
DTYPE_F32, DTYPE_NIBBLE, DTYPE_INT8 = 0, 1, 2
_MAX_NDIM = 8
_CONFIG_KEYS = ("d_model", "n_heads", "d_ff", "experts", "top_k", "layers", "calib_tokens", "seed")


def _unpack_flat(raw: bytes, numel: int) -> np.ndarray:
    b = np.frombuffer(raw, dtype=np.uint8)
    out = np.empty(2 * b.size, dtype=np.uint8)
    out[0::2] = b & 0xF
    out[1::2] = b >> 4
    return out[:numel]


def read_container(path: str):
    """(config dict, tensors dict name -> (dtype code, ndarray)); nibble tensors
    come back as uint8 ids in 0..15.  Same checks and FormatError cases as the
    reference reader (container.py:103-165)."""
    with open(path, "rb") as f:
        data = f.read()
    pos = 0

    def take(n, what):
        nonlocal pos
        if pos + n > len(data):
            raise FormatError(f"truncated container while reading {what}")
        out = data[pos:pos + n]
        pos += n
        return out

    def u32(what):
        return struct.unpack("<I", take(4, what))[0]

    def u64(what):
        return struct.unpack("<Q", take(8, what))[0]

    if take(4, "magic") != MAGIC:
        raise FormatError("bad magic, not a model container")
    version = u32("version")
    if version != VERSION:
        raise FormatError(f"unsupported container version {version}")
    text = take(u64("config length"), "config text")
    try:
        decoded = text.decode("utf-8")
    except UnicodeDecodeError as exc:
        raise FormatError(f"config text is not valid UTF-8: {exc}") from None
    config = {}
    for ln, line in enumerate(decoded.splitlines()):
        if " = " not in line:
            raise FormatError(f"malformed config line {ln + 1}: {line!r}")
        key, value = line.split(" = ", 1)
        if key in config:
            raise FormatError(f"duplicate config key {key!r}")
        config[key] = value
    tensors = {}
    for _ in range(u32("tensor count")):
        name = take(u32("tensor name length"), "tensor name").decode("utf-8")
        if name in tensors:
            raise FormatError(f"duplicate tensor {name!r}")
        code = take(1, f"dtype of tensor {name!r}")[0]
        ndim = u32(f"rank of tensor {name!r}")
        if ndim > _MAX_NDIM:
            raise FormatError(f"tensor {name!r} rank {ndim} exceeds {_MAX_NDIM}")
        dims = tuple(u64(f"dims of tensor {name!r}") for _ in range(ndim))
        numel = int(np.prod(dims, dtype=np.int64)) if dims else 1
        if code == DTYPE_F32:
            arr = np.frombuffer(take(4 * numel, f"payload of tensor {name!r}"), dtype="<f4").reshape(dims)
        elif code == DTYPE_NIBBLE:
            arr = _unpack_flat(take((numel + 1) // 2, f"payload of tensor {name!r}"), numel).reshape(dims)
        elif code == DTYPE_INT8:
            arr = np.frombuffer(take(numel, f"payload of tensor {name!r}"), dtype=np.int8).reshape(dims)
        else:
            raise FormatError(f"tensor {name!r} has unknown dtype code {code}")
        tensors[name] = (code, arr.copy())
    if pos != len(data):
        raise FormatError(f"{len(data) - pos} trailing bytes after last tensor")
    return config, tensors


def _int(config, key):
    if key not in config:
        raise FormatError(f"config key {key!r} missing from container")
    try:
        return int(config[key])
    except ValueError:
        raise FormatError(f"config key {key!r} is not an integer: {config[key]!r}") from None


def site_path(layer: int, site: str, expert: int | None = None) -> str:
    """Tensor names of the container (model.py:104-107)."""
    return f"layer{layer}.{site}" if expert is None else f"layer{layer}.expert{expert}.{site}"


def clustered_site(tensors: dict, name: str):
    """(centroids (d_out, n_groups, K) f32, ids (d_out, d_in) u8, group size)
    of a clustered site, validated like load_model's `grab` (container.py:234-248)."""
    if name + ".centroids" not in tensors:
        if name in tensors:
            raise ConfigError(f"site {name!r} is stored dense; the LUT path needs a clustered site")
        raise FormatError(f"tensor {name!r} missing from container")
    ccode, centroids = tensors[name + ".centroids"]
    if name + ".ids" not in tensors:
        raise FormatError(f"tensor {name + '.ids'!r} missing from container")
    icode, ids = tensors[name + ".ids"]
    if ccode != DTYPE_F32 or icode != DTYPE_NIBBLE:
        raise FormatError(f"clustered site {name!r} has wrong dtype codes")
    if centroids.ndim != 3 or ids.ndim != 2:
        raise FormatError(f"clustered site {name!r} has wrong ranks")
    d_out, n_groups, _ = centroids.shape
    if ids.shape[0] != d_out or n_groups == 0 or ids.shape[1] % n_groups:
        raise FormatError(f"clustered site {name!r} shape mismatch")
    return np.ascontiguousarray(centroids, np.float32), np.ascontiguousarray(ids, np.uint8), ids.shape[1] // n_groups


def moe_layers_from_container(path: str, layers=None, path_kind: str = "auto", prepare_tc: bool = True):
    """One MoELayer per decoder layer (or the given layer indices) from the
    container's router weights and clustered expert codebooks, on the device."""
    from .lutgemm import pack_weights
    from .moe import MoELayer

    config, tensors = read_container(path)
    d, ff, n_exp, top_k = (_int(config, k) for k in ("d_model", "d_ff", "experts", "top_k"))
    n_layers = _int(config, "layers")
    out = []
    for li in (range(n_layers) if layers is None else layers):
        if not 0 <= li < n_layers:
            raise ConfigError(f"layer {li} outside [0, {n_layers})")
        code, w_router = tensors.get(site_path(li, "router"), (None, None))
        if w_router is None:
            raise FormatError(f"tensor {site_path(li, 'router')!r} missing from container")
        if code != DTYPE_F32 or w_router.shape != (d, n_exp):
            raise FormatError(f"router of layer {li} has wrong dtype or shape {w_router.shape}")
        experts = []
        for e in range(n_exp):
            mats = []
            for site, (di, do) in (("gate", (d, ff)), ("up", (d, ff)), ("down", (ff, d))):
                cents, ids, g = clustered_site(tensors, site_path(li, site, e))
                if ids.shape != (do, di):
                    raise FormatError(f"{site_path(li, site, e)!r} has shape {ids.shape}, expected {(do, di)}")
                mats.append(pack_weights(cents, ids, g))
            experts.append(tuple(mats))
        layer = MoELayer(np.ascontiguousarray(w_router, np.float32), experts, top_k, path=path_kind)
        if prepare_tc and path_kind in ("auto", "tc") and d % 128 == 0 and ff % 128 == 0:
            try:
                layer.prepare_tc()
            except Exception:  # shapes outside the tensor-core envelope stay on the fp32 path
                if path_kind == "tc":
                    raise
        out.append(layer)
    return out
