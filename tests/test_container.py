"""CQM1 container reader against a container written by
the reference's own save_model (tests/golden/make_cqm1.py): every expert
codebook and router weight reads back exactly as the reference reads it, and
malformed files raise FormatError like the reference reader."""

import os

import numpy as np
import pytest

from paper_2604_10496_b200.container import clustered_site, read_container, site_path
from paper_2604_10496_b200.errors import ConfigError, FormatError

HERE = os.path.dirname(os.path.abspath(__file__))
PATH = os.path.join(HERE, "golden", "tiny_model.cqm1")


@pytest.fixture(scope="module")
def ref():
    return np.load(os.path.join(HERE, "golden", "tiny_model_ref.npz"))


def test_reads_reference_container_exactly(ref):
    config, tensors = read_container(PATH)
    assert sorted(f"{k}={v}" for k, v in config.items()) == list(ref["config"])
    for li in range(2):
        assert np.array_equal(tensors[site_path(li, "router")][1].view(np.int32), ref[f"router{li}"].view(np.int32))
        for e in range(4):
            for s in ("gate", "up", "down"):
                cents, ids, g = clustered_site(tensors, site_path(li, s, e))
                assert g == int(ref[f"l{li}e{e}{s}_g"])
                assert np.array_equal(ids, ref[f"l{li}e{e}{s}_ids"])
                assert np.array_equal(cents.view(np.int32), ref[f"l{li}e{e}{s}_centroids"].view(np.int32))


def test_dense_site_is_rejected_for_the_lut_path():
    _, tensors = read_container(PATH)
    with pytest.raises(ConfigError):
        clustered_site(tensors, site_path(0, "q"))  # attention weights are stored dense here


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"XQM1" + b[4:], "bad magic"),
    (lambda b: b[:4] + (2).to_bytes(4, "little") + b[8:], "unsupported container version"),
    (lambda b: b[:-3], "truncated"),
    (lambda b: b + b"\0\0", "trailing bytes"),
])
def test_malformed_containers_raise(tmp_path, mutate, msg):
    data = open(PATH, "rb").read()
    bad = tmp_path / "bad.cqm1"
    bad.write_bytes(mutate(data))
    with pytest.raises(FormatError, match=msg):
        read_container(str(bad))
