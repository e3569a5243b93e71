"""ctypes binding of the in-tree C-ABI library ``libfbb200.so``.

The library is the product: there is no Python or CPU fallback for any
operator apply.  If the shared object is missing this module raises at
import time (``build()`` in ``__graft_entry__`` / ``_build.py`` creates it).
"""

import ctypes as C
import os

import numpy as np

from ._build import LIB as _LIB_PATH

FB_OK = 0
FB_ERR_ARG = 1
FB_ERR_CUDA = 2
FB_ERR_OOM = 3
FB_ERR_UNSUPPORTED = 4

KIND = {"mass": 0, "stiffness": 1, "helmholtz": 2, "gradient": 3, "divergence": 4,
        "convection": 5, "curlcurl": 6}

_vp = C.c_void_p
_i64 = C.c_int64
_int = C.c_int
_dbl = C.c_double
_pd = C.POINTER(C.c_double)
_pi64 = C.POINTER(C.c_int64)

# (name, restype, argtypes); every symbol of include/fbb200.h
_SIGS = [
    ("fb_last_error", C.c_char_p, []),
    ("fb_abi_version", _int, []),
    ("fb_launch_count", _i64, []),
    ("fb_restriction_create", _int, [_int, _int, _i64, _i64, _vp, C.POINTER(_vp)]),
    ("fb_restriction_destroy", None, [_vp]),
    ("fb_restriction_ndofs", _i64, [_vp]),
    ("fb_restriction_gather", _int, [_vp, _vp, _vp, _vp]),
    ("fb_restriction_scatter_add", _int, [_vp, _vp, _vp, _vp]),
    ("fb_operator_create", _int, [_int, _vp, _vp, _int, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                  _vp, C.POINTER(_vp)]),
    ("fb_operator_create_geom", _int, [_int, _vp, _vp, _int, _int, _vp, _vp, _vp, _vp, _vp, _vp,
                                       _vp, _dbl, _dbl, C.POINTER(_vp)]),
    ("fb_operator_factor_count", _i64, [_vp]),
    ("fb_set_fast_config", _int, [_int, _int]),
    ("fb_last_fast_launch", _int, [_vp, _vp, _vp]),
    ("fb_set_fast_skip", _int, [_int]),
    ("fb_operator_factors", _int, [_vp, _vp, _i64]),
    ("fb_operator_destroy", None, [_vp]),
    ("fb_operator_apply", _int, [_vp, _vp, _vp, _vp]),
    ("fb_operator_apply_part", _int, [_vp, _vp, _vp, _int, _vp]),
    ("fb_operator_apply_transpose", _int, [_vp, _vp, _vp, _vp]),
    ("fb_operator_device_bytes", _i64, [_vp]),
    ("fb_operator_fast_path", _int, [_vp]),
    ("fb_mask_copy_zero", _int, [_vp, _vp, _i64, _vp, _i64, _vp]),
    ("fb_mask_restore", _int, [_vp, _vp, _vp, _i64, _vp]),
    ("fb_number_dofs_host", _i64, [_int, _int, _i64, _i64, _vp, _vp, _pi64, _pi64]),
    ("fb_dot_partials", _i64, [_i64]),
    ("fb_dot", _int, [_i64, _vp, _vp, _vp, _vp, _vp]),
    ("fb_cg_update", _int, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _int, _vp]),
    ("fb_while_graph_create", _int, [C.POINTER(_vp)]),
    ("fb_while_graph_handle", C.c_ulonglong, [_vp]),
    ("fb_while_graph_begin", _int, [_vp, _vp]),
    ("fb_while_graph_end", _int, [_vp, _vp]),
    ("fb_while_graph_launch", _int, [_vp, _vp]),
    ("fb_while_graph_destroy", None, [_vp]),
    ("fb_cg_check", _int, [C.c_ulonglong, _int, _vp, _vp, _vp, _vp, _int, _vp]),
    ("fb_xpby_dev", _int, [_i64, _vp, _vp, _vp, _vp]),
    ("fb_axpby", _int, [_i64, _dbl, _vp, _dbl, _vp, _vp]),
    ("fb_axpy_dev", _int, [_i64, _vp, _int, _vp, _vp, _vp]),
    ("fb_scalar_div", _int, [_vp, _vp, _vp, _vp]),
    ("fb_xpby_ratio", _int, [_i64, _vp, _vp, _vp, _vp, _vp]),
    ("fb_vmul", _int, [_i64, _vp, _vp, _vp, _vp]),
    ("fb_div_scalar", _int, [_i64, _vp, _dbl, _vp, _vp]),
    ("fb_scale", _int, [_i64, _dbl, _vp, _vp, _vp]),
    ("fb_shift_ratio", _int, [_i64, _vp, _vp, _dbl, _vp, _vp]),
    ("fb_safe_div", _int, [_vp, _vp, _vp, _vp]),
    ("fb_csr_create", _int, [_i64, _i64, _i64, _vp, _vp, _vp, C.POINTER(_vp)]),
    ("fb_csr_destroy", None, [_vp]),
    ("fb_csr_spmv", _int, [_vp, _vp, _vp, _vp]),
    ("fb_csr_residual", _int, [_vp, _vp, _vp, _vp, _vp]),
    ("fb_csr_residual_multi", _int, [_vp, _int, _vp, _vp, _vp, _i64, _vp]),
    ("fb_trisolve_create", _int, [_i64, _vp, _vp, _vp, _int, _int, C.POINTER(_vp)]),
    ("fb_trisolve_destroy", None, [_vp]),
    ("fb_trisolve_solve", _int, [_vp, _vp, _vp, _vp]),
    ("fb_trisolve_levels", _int, [_vp]),
    ("fb_set_trisolve_mode", _int, [_int, _int]),
    ("fb_permute", _int, [_i64, _vp, _vp, _vp, _int, _vp]),
    ("fb_ilu0_factor_host", _i64, [_i64, _vp, _vp, _vp]),
    ("fb_lor_assemble_host", _i64, [_int, _int, _i64, _i64, _vp, _vp, _vp, _int, _dbl, _dbl, _i64,
                                    _vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp)]),
    ("fb_host_free", None, [_vp]),
    ("fb_blockilu_create", _int, [_i64, _int, _vp, _vp, _vp, _vp, _vp, C.POINTER(_vp)]),
    ("fb_blockilu_info", _int, [_vp, _vp, _vp, _vp, _vp]),
    ("fb_blockilu_sweep_kind", _int, [_vp]),
    ("fb_blockilu_apply_add", _int, [_vp, _int, _vp, _vp, _vp]),
    ("fb_blockilu_destroy", None, [_vp]),
    ("fb_blockilu_apply", _int, [_vp, _int, _vp, _vp, _vp]),
    ("fb_dense_mv", _int, [_i64, _vp, _vp, _vp, _vp]),
    ("fb_lor_assemble_box", _int, [_int, _vp, _vp, _vp, _vp, _int, _dbl, _dbl, _int,
                                   C.POINTER(_vp)]),
    ("fb_lor_assemble_box_rows", _int, [_int, _vp, _vp, _vp, _vp, _int, _dbl, _dbl, _int, _i64,
                                        _i64, C.POINTER(_vp)]),
    ("fb_csr_pin", _int, [_vp, _i64]),
    ("fb_csr_info", _int, [_vp, _pi64, _pi64, _pi64]),
    ("fb_csr_download", _int, [_vp, _vp, _vp, _vp]),
    ("fb_set_blockilu_packed", _int, [_int]),
    ("fb_blockilu_create_csr", _int, [_vp, _i64, _vp, _pi64, C.POINTER(_vp)]),
    ("fb_transfer_create", _int, [_vp, _vp, _vp, _int, _vp, _vp, C.POINTER(_vp)]),
    ("fb_transfer_destroy", None, [_vp]),
    ("fb_transfer_set_periodic", _int, [_vp, _int, _i64, _i64, _i64]),
    ("fb_transfer_set_origin", _int, [_vp, _i64, _i64, _i64]),
    ("fb_index_add", _int, [_i64, _vp, _vp, _vp, _vp]),
    ("fb_transfer_prolong", _int, [_vp, _vp, _vp, _vp]),
    ("fb_transfer_prolong_add", _int, [_vp, _vp, _vp, _vp]),
    ("fb_transfer_restrict", _int, [_vp, _vp, _vp, _vp]),
    ("fb_set_blockilu_pipeline", _int, [_int, _int]),
]

SYMBOLS = [s[0] for s in _SIGS]


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(
            f"{_LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = C.CDLL(_LIB_PATH)
    for name, res, args in _SIGS:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
LIB_PATH = _LIB_PATH


def check(rc):
    """Map a C status to the reference's exception types."""
    if rc == FB_OK:
        return
    msg = (lib.fb_last_error() or b"").decode()
    if rc == FB_ERR_ARG:
        raise ValueError(msg)
    if rc == FB_ERR_OOM:
        raise MemoryError(msg)
    raise RuntimeError(f"fbb200 error {rc}: {msg}")


def ptr(a):
    """Raw address of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def host_f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def host_i64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int64)
