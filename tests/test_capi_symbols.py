"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/fastmaxent.h
declares, and rejects bad arguments before touching the device (no compute calls here)."""
import ctypes as C
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fastmaxent.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fm_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header_symbols():
    from paper_2509_13230_b200 import build as B
    B.build()
    lib = C.CDLL(B.LIB)
    names = _declared()
    assert {"fm_sort_plan", "fm_sample_ubcm", "fm_sample_ecm", "fm_free"} <= set(names)
    for nm in names:
        assert hasattr(lib, nm), nm
    from paper_2509_13230_b200 import fastmaxent as fm
    assert set(fm.SYMBOLS) == set(names)
    assert fm.abi_version() == 1


def test_argument_validation_without_device():
    from paper_2509_13230_b200 import fastmaxent as fm
    lib = fm.lib
    h = C.c_void_p()
    x = (C.c_double * 1)(1.0)
    assert lib.fm_sort_plan(0, 1, C.cast(x, C.c_void_p), None, 0, None, C.byref(h)) == fm.FM_ERR_INVALID
    assert b"outside" in lib.fm_last_error()
    assert lib.fm_sort_plan(7, 4, C.cast(x, C.c_void_p), None, 0, None, C.byref(h)) == fm.FM_ERR_INVALID
    assert lib.fm_sort_plan(1, 4, C.cast(x, C.c_void_p), None, 0, None, C.byref(h)) == fm.FM_ERR_INVALID  # ECM w/o y
    assert lib.fm_sort_plan(0, 4, C.cast(x, C.c_void_p), None, 5, None, C.byref(h)) == fm.FM_ERR_INVALID  # S < 8
    st = fm._Edges()
    assert lib.fm_sample_ubcm(None, 1, 0, 1, None, C.byref(st)) == fm.FM_ERR_STATE
    # fm_expected_degrees: argument checks come before any device access
    assert lib.fm_expected_degrees(0, 0, C.cast(x, C.c_void_p), None, None, 0, None, None, None, None,
                                   None) == fm.FM_ERR_INVALID
    assert lib.fm_expected_degrees(0, 1, C.cast(x, C.c_void_p), C.cast(x, C.c_void_p), None, 1, None, None,
                                   None, None, None) == fm.FM_ERR_INVALID  # UBCM takes no y
    assert lib.fm_expected_degrees(1, 1, C.cast(x, C.c_void_p), None, None, 1, None, None, None, None,
                                   None) == fm.FM_ERR_INVALID  # ECM needs y
    lib.fm_free(None)  # no-op


def test_no_oracle_in_product():
    """The product package never imports, links or calls oracle/ (and vice versa)."""
    bad = re.compile(r"(^\s*(from|import)\s+oracle)|fmo\.h|libfmo|\bfmo_[a-z]", re.M)
    pkg = os.path.join(ROOT, "paper_2509_13230_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                assert not bad.search(open(os.path.join(dirpath, f)).read()), f
    back = re.compile(r"fastmaxent\.h|libfastmaxent|^\s*(from|import)\s+paper_2509_13230_b200\.(fastmaxent|build)", re.M)
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".c", ".h", ".py")):
            assert not back.search(open(os.path.join(ROOT, "oracle", f)).read()), f
