"""CPU checks of the C-ABI boundary: the in-tree library exists, loads, and exports
every symbol that include/*.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in ("omniseg.h", "omniseg_debug.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(omniseg_[a-z_]+)\s*\(", src):
            names.add(m.group(1))
    return names


def test_headers_declare_the_north_star_calls():
    names = declared_symbols()
    assert {"omniseg_create", "omniseg_segment_slide", "omniseg_segment_band", "omniseg_destroy"} <= names


def test_library_exports_every_declared_symbol():
    from paper_2305_14566_b200 import build, lib
    path = build.build(verbose=False)
    so = ctypes.CDLL(path)
    missing = [n for n in sorted(declared_symbols()) if not hasattr(so, n)]
    assert not missing, missing
    assert set(lib.SYMBOLS) == declared_symbols()


def test_binding_fails_loudly_without_library(tmp_path):
    from paper_2305_14566_b200 import lib
    saved = lib._lib
    lib._lib = None
    try:
        with pytest.raises(lib.OmnisegError):
            lib.load(str(tmp_path / "nope.so"))
    finally:
        lib._lib = saved


def test_band_rows_helper_arithmetic():
    """omniseg_band_rows is pure arithmetic (no GPU): owned canvas rows of a band."""
    from paper_2305_14566_b200 import lib
    lib.load(lib.LIB_PATH) if os.path.exists(lib.LIB_PATH) else pytest.skip("library not built")
    # H=1000, pad=64, f=1: band [0, 512) owns canvas rows [0, 448); [512, 1152) owns [448, 1000)
    assert lib.band_rows(1000, 0, 512, 64, 1) == (0, 448)
    assert lib.band_rows(1000, 512, 1152, 64, 1) == (448, 1000)
    assert lib.band_rows(1000, 512, 1152, 64, 4) == (112, 250)


def test_no_oracle_import_in_product():
    """The product package never imports the oracle."""
    pkg = os.path.join(ROOT, "paper_2305_14566_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                s = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", s).replace("oracle_", ""), f


@pytest.mark.parametrize("arch, msg", [
    ("levels=5;base=32;head=8;ncls=6;scale_codes=5,10,20,40;slide_mag=40;dtype=fp16f8;batch=0", "batch"),
    ("levels=5;base=32;head=8;ncls=6;scale_codes=5,10,20,40;slide_mag=40;dtype=fp16f8;batch=x", "bad integer"),
    ("levels=5;base=32;nonsense", "key=value"),
    ("levels=5;base=1024;head=8;ncls=6;scale_codes=5,10,20,40;slide_mag=40;dtype=fp16f8;batch=64", "base must"),
    ("levels=5;base=32;head=4;ncls=6;scale_codes=5,10,20,40;slide_mag=40;dtype=fp16f8;batch=64", "head must be 8"),
    ("levels=5;base=32;head=8;ncls=6;scale_codes=5,10,20,40;slide_mag=40;dtype=fp16f8;color=1", "unknown key"),
    ("levels=5;base=32;head=8;ncls=6;scale_codes=5,10,20,40;slide_mag=40;dtype=fp16f8;batch=8;grp=9", "grp must"),
    ("levels=5;base=32;head=8;ncls=6;scale_codes=5,10,20,40;slide_mag=40;dtype=fp16f8;grp=2;glev=0", "glev must"),
    ("levels=5;base=32;head=8;ncls=6;scale_codes=5,10,20,40;slide_mag=40;dtype=fp16f8;hrm=1", "unknown key"),
])
def test_create_rejects_bad_arch_strings_before_touching_the_device(arch, msg):
    """omniseg_create parses and validates the arch string first: a bad one returns NULL with
    a message (no GPU needed to see it)."""
    from paper_2305_14566_b200 import Omniseg, lib
    lib.load(lib.LIB_PATH) if os.path.exists(lib.LIB_PATH) else pytest.skip("library not built")
    with pytest.raises(lib.OmnisegError, match=msg):
        Omniseg(arch, np.zeros(4, np.float32))
