"""Device vector kernels (Krylov building blocks) and device sparse objects.

Thin Python handles over the C ABI (include/fbb200.h): deterministic dots,
axpy-style updates with device-resident scalars, CSR SpMV and sync-free
triangular solves.  All operands are CUDA float64 tensors; nothing here
computes on the host.
"""

import ctypes as C
import threading

import numpy as np
import torch

from . import _lib
from . import device as dev


def _st(stream=None):
    return dev.stream_handle() if stream is None else stream


class Workspace:
    """Scratch for reductions: partial sums sized for the largest vector."""

    def __init__(self, n):
        self.n = n
        self.partial = dev.empty(int(_lib.lib.fb_dot_partials(max(n, 1))))
        self.scalars = dev.zeros(16)

    def ensure(self, n):
        if n > self.n:
            self.__init__(n)


_WS = {}


def workspace(n):
    # per device AND per host thread: the in-process multi-rank tests drive
    # several ranks from threads, which must not share reduction scratch
    key = (torch.cuda.current_device(), threading.get_ident())
    ws = _WS.get(key)
    if ws is None:
        ws = _WS[key] = Workspace(n)
    ws.ensure(n)
    return ws


def dot_into(x, y, out, stream=None):
    """out[0] = x . y (deterministic; out is a 1-element device tensor view)."""
    n = x.shape[0]
    ws = workspace(n)
    _lib.check(_lib.lib.fb_dot(n, x.data_ptr(), y.data_ptr(), ws.partial.data_ptr(),
                               out.data_ptr(), _st(stream)))
    return out


def dot(x, y):
    out = dev.empty(1)
    dot_into(x, y, out)
    return out


def axpby(a, x, b, y, stream=None):
    """y = a*x + b*y (host scalars)."""
    _lib.check(_lib.lib.fb_axpby(y.shape[0], float(a), x.data_ptr(), float(b), y.data_ptr(),
                                 _st(stream)))
    return y


def axpy_dev(alpha, x, y, sign=1, stream=None):
    """y = y + sign * alpha[0] * x with alpha on the device."""
    _lib.check(_lib.lib.fb_axpy_dev(y.shape[0], alpha.data_ptr(), int(sign), x.data_ptr(),
                                    y.data_ptr(), _st(stream)))
    return y


def cg_update(rz, pAp, alpha, p, Ap, x, r, update_r=True, stream=None):
    """alpha = rz/pAp (0 if pAp <= 0); x += alpha p; r -= alpha Ap (fused)."""
    _lib.check(_lib.lib.fb_cg_update(x.shape[0], rz.data_ptr(), pAp.data_ptr(), alpha.data_ptr(),
                                     p.data_ptr(), Ap.data_ptr(), x.data_ptr(), r.data_ptr(),
                                     int(bool(update_r)), _st(stream)))
    return x


def safe_div(num, den, out, stream=None):
    _lib.check(_lib.lib.fb_safe_div(num.data_ptr(), den.data_ptr(), out.data_ptr(), _st(stream)))
    return out


def xpby_ratio(z, num, den, p, stream=None):
    """p = z + (num/den) * p."""
    _lib.check(_lib.lib.fb_xpby_ratio(p.shape[0], z.data_ptr(), num.data_ptr(), den.data_ptr(),
                                      p.data_ptr(), _st(stream)))
    return p


def scale(a, x, y, stream=None):
    """y = a * x."""
    _lib.check(_lib.lib.fb_scale(x.shape[0], float(a), x.data_ptr(), y.data_ptr(), _st(stream)))
    return y


def div_scalar(x, s, y, stream=None):
    """y = x / s."""
    _lib.check(_lib.lib.fb_div_scalar(x.shape[0], x.data_ptr(), float(s), y.data_ptr(), _st(stream)))
    return y


def shift_ratio(x, num, den, y, stream=None):
    """y = x - num[0]/den."""
    _lib.check(_lib.lib.fb_shift_ratio(x.shape[0], x.data_ptr(), num.data_ptr(), float(den),
                                       y.data_ptr(), _st(stream)))
    return y


def vmul(d, x, y, stream=None):
    _lib.check(_lib.lib.fb_vmul(x.shape[0], d.data_ptr(), x.data_ptr(), y.data_ptr(), _st(stream)))
    return y


def copy(x, y, stream=None):
    """y = x (a 1.0 * x scale: never reads y, so uninitialised y is fine)."""
    _lib.check(_lib.lib.fb_scale(x.shape[0], 1.0, x.data_ptr(), y.data_ptr(), _st(stream)))
    return y


def permute(idx, src, dst, scatter=False, stream=None):
    _lib.check(_lib.lib.fb_permute(idx.shape[0], idx.data_ptr(), src.data_ptr(), dst.data_ptr(),
                                   int(scatter), _st(stream)))
    return dst


class DeviceCSR:
    """A scipy CSR matrix on the device; y = A x in scipy's summation order."""

    def __init__(self, A):
        A = A.tocsr()
        A.sort_indices()
        self.shape = A.shape
        ip = np.ascontiguousarray(A.indptr, dtype=np.int64)
        ix = np.ascontiguousarray(A.indices, dtype=np.int64)
        dv = np.ascontiguousarray(A.data, dtype=np.float64)
        dev.device()
        h = C.c_void_p()
        _lib.check(_lib.lib.fb_csr_create(A.shape[0], A.shape[1], A.nnz, _lib.ptr(ip), _lib.ptr(ix),
                                          _lib.ptr(dv), C.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None and _lib.lib is not None:
            _lib.lib.fb_csr_destroy(h)

    def apply_into(self, x, y, stream=None):
        _lib.check(_lib.lib.fb_csr_spmv(self.handle, x.data_ptr(), y.data_ptr(), _st(stream)))
        return y

    def residual_into(self, b, x, y, stream=None):
        """y = b - A x."""
        _lib.check(_lib.lib.fb_csr_residual(self.handle, b.data_ptr(), x.data_ptr(), y.data_ptr(),
                                            _st(stream)))
        return y

    def residual_multi_into(self, nv, stride, b, x, y, stream=None):
        """y_j = b_j - A x_j for nv vectors at a common stride (one matrix read;
        device-assembled matrices only)."""
        _lib.check(_lib.lib.fb_csr_residual_multi(self.handle, int(nv), b.data_ptr(), x.data_ptr(),
                                                  y.data_ptr(), int(stride), _st(stream)))
        return y


class TriSolve:
    """Sparse triangular solve on the device (sync-free, one launch)."""

    def __init__(self, T, lower, unit_diag):
        T = T.tocsr()
        T.sort_indices()
        ip = np.ascontiguousarray(T.indptr, dtype=np.int64)
        ix = np.ascontiguousarray(T.indices, dtype=np.int64)
        dv = np.ascontiguousarray(T.data, dtype=np.float64)
        self.n = T.shape[0]
        dev.device()
        h = C.c_void_p()
        _lib.check(_lib.lib.fb_trisolve_create(self.n, _lib.ptr(ip), _lib.ptr(ix), _lib.ptr(dv),
                                               int(bool(lower)), int(bool(unit_diag)), C.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None and _lib.lib is not None:
            _lib.lib.fb_trisolve_destroy(h)

    def solve_into(self, b, x, stream=None):
        _lib.check(_lib.lib.fb_trisolve_solve(self.handle, b.data_ptr(), x.data_ptr(), _st(stream)))
        return x


def ilu0_factor_host(indptr, indices, data):
    """In-place ILU(0) on sorted CSR arrays (C++); -1 or the failing row."""
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    ix = np.ascontiguousarray(indices, dtype=np.int64)
    if data.dtype != np.float64 or not data.flags.c_contiguous:
        raise ValueError("data must be a contiguous float64 array (factored in place)")
    return int(_lib.lib.fb_ilu0_factor_host(ip.shape[0] - 1, _lib.ptr(ip), _lib.ptr(ix),
                                            _lib.ptr(data)))
