"""C ABI checks that need no GPU: the library loads, exports every symbol
include/sfft_b200.h declares, and its host-only entry points (hyperbolic
cross) reproduce the reference's golden outputs."""

import ctypes
import os
import re

import numpy as np

from conftest import ROOT, golden


def _declared():
    text = open(os.path.join(ROOT, "include", "sfft_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sfftb_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2006_13053_b200 import _native

    so = ctypes.CDLL(_native.LIB_PATH)
    names = _declared()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, missing
    # and the Python binding table covers the header exactly
    assert sorted(_native._SIGS) == names


def test_version_and_error_plumbing():
    from paper_2006_13053_b200 import _native

    assert "sm_100a" in _native.version()
    assert isinstance(_native.lib().sfftb_last_error(), bytes)


def test_plugin_backend_name():
    import paper_2006_13053_b200 as pkg

    assert pkg.kernel_backend == "cuda"


def test_hc_matches_reference_golden():
    from paper_2006_13053_b200 import _kernels

    for case in golden("hc_cases.json"):
        w = np.array(case["w"])
        assert _kernels.hc_count(case["d"], float(case["N"]), w) == case["count"]
        rows = _kernels.hc_enumerate(case["d"], float(case["N"]), w)
        assert np.array_equal(rows, np.array(case["rows"], dtype=np.int64).reshape(-1, case["d"]))


def test_hyperbolic_cross_paper_counts():
    from paper_2006_13053_b200 import hyperbolic_cross

    # PAPER.md table values quoted in SURVEY section 4
    assert hyperbolic_cross(3, 4, count_only=True) == 225


def test_stage_descriptor_layout_matches_header(tmp_path):
    """_stage.StageDesc mirrors sfftb_stage_t field for field (offsets, size)."""
    import ctypes
    import subprocess

    from paper_2006_13053_b200._stage import StageDesc

    names = [f[0] for f in StageDesc._fields_]
    src = tmp_path / "layout.c"
    src.write_text("#include <stdio.h>\n#include <stddef.h>\n#include \"sfft_b200.h\"\n"
                   "int main(void){printf(\"%zu\\n\", sizeof(sfftb_stage_t));\n" +
                   "".join(f"printf(\"%zu\\n\", offsetof(sfftb_stage_t, {n}));\n" for n in names)
                   + "return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    out = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    assert out[0] == ctypes.sizeof(StageDesc)
    assert out[1:] == [getattr(StageDesc, n).offset for n in names]
