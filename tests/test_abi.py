"""CPU tests of the boundary: the C-ABI library loads and exports every symbol
include/rhosvd.h declares, and the binding's host logic (no compute calls)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "rhosvd.h")


def header_functions():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = re.findall(r"\b(rhosvd_[a-z0-9_]+)\s*\(", txt)
    return sorted(set(n for n in names if n not in ("rhosvd_allreduce_fn",)))


@pytest.fixture(scope="module")
def lib():
    from paper_2201_12663_b200 import rhosvd
    if not os.path.exists(rhosvd.LIB_PATH):
        from paper_2201_12663_b200.build import build
        build()
    return rhosvd.lib()


def test_library_exports_every_header_symbol(lib):
    names = header_functions()
    assert len(names) >= 19
    for nm in names:
        assert hasattr(lib, nm), nm
    from paper_2201_12663_b200 import rhosvd
    assert sorted(rhosvd.EXPORTED) == names


def test_opts_default_and_struct_layout(lib):
    from paper_2201_12663_b200 import rhosvd
    o = rhosvd.Opts()
    lib.rhosvd_opts_default(ctypes.byref(o))
    assert o.rank_mode == rhosvd.RHOSVD_EPS and o.oversample == 16 and o.block0 == 0
    assert o.refine_steps == 1 and o.flags == rhosvd.RHOSVD_F_SIGN_FIX
    assert ctypes.sizeof(rhosvd.Opts) == 56
    o2 = rhosvd.make_opts(ranks=(3, 4, 5))
    assert o2.rank_mode == rhosvd.RHOSVD_FIXED_RANK and list(o2.r) == [3, 4, 5]
    with pytest.raises(ValueError):
        rhosvd.make_opts()


def test_argument_validation_without_gpu(lib):
    """EINVAL paths return before touching the device."""
    from paper_2201_12663_b200 import rhosvd
    o = rhosvd.make_opts(eps=1e-3)
    h = ctypes.c_void_p()
    P = ctypes.c_void_p
    # n < 1
    s = lib.rhosvd_c2t(P(0), P(0), P(0), 1, P(0), 0, 0, ctypes.byref(o), None, None, ctypes.byref(h))
    assert s == -1 and h.value is None
    # ldu < n
    s = lib.rhosvd_c2t(P(8), P(8), P(8), 3, P(8), 5, 2, ctypes.byref(o), None, None, ctypes.byref(h))
    assert s == -1
    # eps outside (0, 1)
    o.eps = 1.5
    s = lib.rhosvd_c2t(P(8), P(8), P(8), 5, P(8), 5, 2, ctypes.byref(o), None, None, ctypes.byref(h))
    assert s == -1 and b"eps" in lib.rhosvd_last_error()
    # fixed rank < 1
    o2 = rhosvd.make_opts(ranks=(0, 1, 1))
    s = lib.rhosvd_c2t(P(8), P(8), P(8), 5, P(8), 5, 2, ctypes.byref(o2), None, None, ctypes.byref(h))
    assert s == -1
    assert lib.rhosvd_version().startswith(b"rhosvd-b200")


def test_report_struct_size():
    from paper_2201_12663_b200 import rhosvd
    # 3+3+1+1+1+1+3 doubles, 3*4 int32 + int64 + 16 doubles + 3 doubles + int32 (+pad)
    assert ctypes.sizeof(rhosvd.Report) == 8 * 13 + 4 * 12 + 8 + 8 * 16 + 8 * 3 + 4 + 4 * 3


def test_no_oracle_import_in_product():
    """The product package never imports oracle/ (no CPU fallback path)."""
    pkg = os.path.join(ROOT, "paper_2201_12663_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
