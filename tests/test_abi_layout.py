"""The ctypes mirror of include/cq_b200.h (paper_2604_10496_b200/_lib.py) against
the header itself, compiled here with gcc: every field offset and the size of
cq_expert_site / cq_moe_desc, and the enum values the Python side hard-codes
(workspace buffer order, tensor-core layouts, paths, flags).  A struct edit on
one side without the other fails here, on CPU, instead of as garbage on a GPU."""

import ctypes
import os
import shutil
import subprocess

import pytest

from paper_2604_10496_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INCLUDE = os.path.join(ROOT, "include")

pytestmark = pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")


def _c_values(tmp_path, exprs):
    """Evaluate integer C expressions (sizeof / offsetof / enum constants) against the header."""
    body = "\n".join(f'    printf("%lld\\n", (long long)({e}));' for e in exprs)
    src = tmp_path / "abi.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "cq_b200.h"\nint main(void) {\n'
                   + body + "\n    return 0;\n}\n")
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-std=c11", "-I", INCLUDE, str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    return [int(v) for v in out]


@pytest.mark.parametrize("py,c", [(_lib.ExpertSite, "cq_expert_site"), (_lib.MoEDesc, "cq_moe_desc")])
def test_struct_layout_matches_header(tmp_path, py, c):
    names = [f[0] for f in py._fields_]
    exprs = [f"sizeof({c})"] + [f"offsetof({c}, {n})" for n in names]
    got = _c_values(tmp_path, exprs)
    assert got[0] == ctypes.sizeof(py)
    assert got[1:] == [getattr(py, n).offset for n in names]


def test_enums_match_header(tmp_path):
    ws = ["CQ_WS_" + n.upper() for n in _lib.WS_NAMES]
    layouts = ["CQ_TC_UMMA128U", "CQ_TC_UMMA128U8"]
    paths = ["CQ_PATH_AUTO", "CQ_PATH_F32", "CQ_PATH_TC", "CQ_PATH_ORDERED"]
    got = _c_values(tmp_path, ["CQ_WS_COUNT_"] + ws + layouts + paths + ["CQ_FLAG_KEEP_HIDDEN"])
    assert got[0] == len(_lib.WS_NAMES)
    assert got[1:1 + len(ws)] == list(range(len(ws)))
    i = 1 + len(ws)
    assert got[i:i + 2] == [_lib.TC_LAYOUTS[k] for k in ("umma128u", "umma128u8")]
    assert got[i + 2:i + 6] == [_lib.CQ_PATH_AUTO, _lib.CQ_PATH_F32, _lib.CQ_PATH_TC, _lib.CQ_PATH_ORDERED]
    assert got[i + 6] == _lib.FLAG_KEEP_HIDDEN
