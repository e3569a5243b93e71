"""CPU: the C-ABI library loads and exports every symbol include/fbb200.h
declares; host-only entry points behave."""

import ctypes as C
import os
import re

import numpy as np

from paper_1910_03032_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if not fn.endswith(".h"):
            continue
        text = open(os.path.join(ROOT, "include", fn)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(fb_[a-z0-9_]+)\s*\(", text):
            names.add(m.group(1))
    return names


def test_library_is_in_tree_and_loads():
    assert os.path.dirname(_lib.LIB_PATH).startswith(ROOT)
    assert _lib.lib.fb_abi_version() == 1


def test_exports_every_declared_symbol():
    declared = header_functions()
    assert declared, "no declarations parsed"
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in sorted(declared) if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes table binds exactly the declared API
    assert declared == set(_lib.SYMBOLS)


def test_host_numbering_entry_point_and_errors():
    elems = np.array([[0, 1, 2, 3]], dtype=np.int64)
    out = np.empty((1, 9), dtype=np.int64)
    ne, nf = C.c_int64(), C.c_int64()
    nd = _lib.lib.fb_number_dofs_host(2, 2, 1, 4, _lib.ptr(elems), _lib.ptr(out), C.byref(ne),
                                      C.byref(nf))
    assert nd == 9 and ne.value == 4
    # vertices first, then the 4 edges in local-edge order, then the interior
    assert list(out[0]) == [0, 4, 1, 6, 8, 7, 2, 5, 3]  # flowbench FESpace on a 1x1 mesh
    bad = _lib.lib.fb_number_dofs_host(5, 2, 1, 4, _lib.ptr(elems), _lib.ptr(out), None, None)
    assert bad == -_lib.FB_ERR_ARG
    assert b"dim" in _lib.lib.fb_last_error()


def test_dot_partials_sizes():
    assert _lib.lib.fb_dot_partials(0) == 1
    assert _lib.lib.fb_dot_partials(4096) == 1
    assert _lib.lib.fb_dot_partials(4097) == 2
