"""C-ABI library checks that need no GPU: the library loads, exports every symbol include/podp.h declares, and
argument validation returns status codes (never aborts) before touching a device."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2307_05590_b200 as pb
from paper_2307_05590_b200 import podp as P
import podp_inputs as g

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    return pb.load_library()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "podp.h")).read()
    return sorted(set(re.findall(r"^\s*(?:podp_status|int32_t|const char \*)\s*(podp_\w+)\s*\(", txt, re.M)))


def test_exports_every_declared_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(P.EXPORTED) == syms


def test_version_and_null_safety(lib):
    assert b"sm_100a" in lib.podp_version()
    assert lib.podp_destroy(None) == 0
    assert lib.podp_n_obj(None) == 0 and lib.podp_r(None) == 0


def test_eval_select_null_ctx(lib):
    st = lib.podp_eval(None, None, 10, None, None, None, None, None, 0, None)
    assert st == 1 and b"ctx" in lib.podp_last_error()
    st = lib.podp_select(None, None, None, 0, None, 0, 2, 0.0, None, None, None, None, None, None)
    assert st == 1


def _create_status(lib, o):
    keep = []
    st = P._marshal(o, keep)
    h = ctypes.c_void_p()
    return lib.podp_create(ctypes.byref(st), 0, None, ctypes.byref(h)), lib.podp_last_error().decode()


def test_validation_codes(lib):
    o = g.make_operators(8)
    bad = o.copy(); bad.nu = -1.0
    assert _create_status(lib, bad)[0] == 1
    bad = o.copy(); bad.alpha_lb = 0.0
    assert _create_status(lib, bad)[0] == 1
    bad = o.copy(); bad.K = bad.K.copy(); bad.K[0, 1] += 0.5          # corrupted entry -> not Hermitian
    st, msg = _create_status(lib, bad)
    assert st == 6 and "K" in msg
    bad = o.copy(); bad.G = bad.G.copy(); bad.G[3, 9] += 1j
    assert _create_status(lib, bad)[0] == 6
    bad = o.copy(); bad.b1 = bad.b1.copy(); bad.b1[2, 1] = np.nan
    assert _create_status(lib, bad)[0] == 5
    bad = o.copy(); bad.S = bad.S.copy(); bad.S[0, 1] += 1.0
    assert _create_status(lib, bad)[0] == 1


def test_r_out_of_range(lib):
    o = g.make_operators(8)
    keep = []
    st = P._marshal(o, keep)
    st.r = 0
    h = ctypes.c_void_p()
    assert lib.podp_create(ctypes.byref(st), 0, None, ctypes.byref(h)) == 1
    st.r = P.R_MAX + 1
    assert lib.podp_create(ctypes.byref(st), 0, None, ctypes.byref(h)) == 1


def test_batch_mixed_r_rejected(lib):
    keep = []
    arr = (P.podp_operators * 2)(P._marshal(g.make_operators(8), keep), P._marshal(g.make_operators(10), keep))
    h = ctypes.c_void_p()
    assert lib.podp_create_batch(2, arr, 0, None, ctypes.byref(h)) == 1
    assert b"differs" in lib.podp_last_error()


def test_product_does_not_import_oracle():
    """The product package must never reach into oracle/ (test infrastructure only)."""
    pkg = os.path.join(ROOT, "paper_2307_05590_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("oracle/", ""), f
