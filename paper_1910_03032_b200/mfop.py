"""Matrix-free operators on the B200: drop-in for the reference's ``mfop``.

Same classes, constructor signatures, attributes and error behaviour as the
reference (mfop.py:98-452): ``MassOperator(space, geom)``,
``StiffnessOperator(space, geom, nu)``, ``HelmholtzOperator(space, geom, c,
nu)``, ``GradientOperator(vspace, pspace, geom)`` (+ ``apply_transpose``),
``DivergenceOperator(vspace, pspace, geom)``, ``ConstrainedOperator(op,
dofs)`` and the ``setup(kind, ...)`` factory.  ``space`` / ``geom`` may be the
reference's own ``FESpace`` / ``GeometricFactors`` or this package's
(``spaces.FESpace``, ``geometry.GeometricFactors`` / ``DeviceGeometry``).

``apply`` runs on the GPU through the C ABI (include/fbb200.h).  A numpy
operand is copied to the device and the result copied back (numpy in, numpy
out, as the reference's tests expect); a CUDA float64 tensor stays on the
device and a CUDA tensor is returned.  ``apply_into(x, y)`` writes into a
preallocated device vector (no allocation; what the solvers use).  There
is no CPU path: without the CUDA library or a GPU the constructors raise.
"""

import ctypes as C
import time
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import device as dev
from .quadrature import build_eval_matrices

_SYM_PAIRS = {2: [(0, 0), (0, 1), (1, 1)], 3: [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]}


class MemoryCapError(RuntimeError):
    """Raised when an assembled matrix would exceed the configured cap."""


# -- device element restrictions, one per space object ------------------------

class Restriction:
    """Owner of the device L->E map / transposed map of one space."""

    def __init__(self, space):
        ed = np.ascontiguousarray(space.element_dofs, dtype=np.int64)
        h = C.c_void_p()
        _lib.check(_lib.lib.fb_restriction_create(space.dim, space.p, ed.shape[0],
                                                  space.ndofs_scalar, _lib.ptr(ed), C.byref(h)))
        self.handle = h
        self.ndofs = space.ndofs_scalar
        self.ne = ed.shape[0]
        self.nloc = ed.shape[1]

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None and _lib.lib is not None:
            _lib.lib.fb_restriction_destroy(self.handle)
            self.handle = None

    def gather(self, x):
        """E-array (ne, nloc) of a scalar device vector (fespace.py:282-284)."""
        xd, host = dev.DeviceIn.get(x)
        out = dev.empty(self.ne * self.nloc)
        _lib.check(_lib.lib.fb_restriction_gather(self.handle, xd.data_ptr(), out.data_ptr(),
                                                  dev.stream_handle()))
        out = out.view(self.ne, self.nloc)
        return dev.to_host(out) if host else out

    def scatter_add(self, xloc):
        """Deterministic E->L sum, bitwise np.bincount (fespace.py:286-292)."""
        xd, host = dev.DeviceIn.get(xloc)
        out = dev.empty(self.ndofs)
        _lib.check(_lib.lib.fb_restriction_scatter_add(self.handle, xd.data_ptr(),
                                                       out.data_ptr(), dev.stream_handle()))
        return dev.to_host(out) if host else out


_RESTRICTIONS = weakref.WeakKeyDictionary()


def restriction(space):
    dev.device()
    try:
        r = _RESTRICTIONS.get(space)
    except TypeError:
        r = None
    if r is None:
        r = Restriction(space)
        try:
            _RESTRICTIONS[space] = r
        except TypeError:
            pass
    return r


# -- factors (host formulas of mfop.py:115-152) -------------------------------

@dataclass
class QPointFactors:
    wdet: np.ndarray = None
    stiff: np.ndarray = None
    grad: np.ndarray = None


def _mass_factor(geom):
    return geom.detj * geom.w[None, :]


def _stiffness_factor(geom, nu):
    d = geom.jinv.shape[-1]
    wdet = _mass_factor(geom)
    out = np.empty(wdet.shape + (len(_SYM_PAIRS[d]),))
    for k, (a, b) in enumerate(_SYM_PAIRS[d]):
        s = np.zeros_like(wdet)
        for m in range(d):
            s += geom.jinv[..., a, m] * geom.jinv[..., b, m]
        out[..., k] = nu * wdet * s
    return out


def _grad_factor(geom):
    wdet = _mass_factor(geom)
    return wdet[..., None, None] * np.swapaxes(geom.jinv, -1, -2)


def _num_elements(geom):
    if hasattr(geom, "num_elements"):
        return geom.num_elements
    return geom.xq.shape[0]


def _check_rule_match(space, geom):
    if _num_elements(geom) != space.mesh.num_elements:
        raise ValueError("geometric factors were built for a different mesh")


def _eval_matrices(space, points):
    basis = space.basis
    if hasattr(basis, "eval_matrices_at"):
        B, D = basis.eval_matrices_at(points)
    else:
        B, D = build_eval_matrices(basis.nodes, points)
    return np.ascontiguousarray(B, dtype=np.float64), np.ascontiguousarray(D, dtype=np.float64)


def _is_device_geom(geom):
    # type check first: hasattr(DeviceGeometry, "detj") would materialise the
    # host factors through the lazy property
    return type(geom).__name__ == "DeviceGeometry" or not hasattr(geom, "detj")


# -- operators -----------------------------------------------------------------

class Operator:
    """A linear map with ``shape`` and ``apply`` (mfop.py:98-113)."""

    shape = None

    def apply(self, x):
        raise NotImplementedError

    def mult(self, x):
        return self.apply(x)

    def __call__(self, x):
        return self.apply(x)

    def __matmul__(self, x):
        if (isinstance(x, np.ndarray) or isinstance(x, torch.Tensor)) and x.ndim == 1:
            return self.apply(x)
        return NotImplemented


class _DeviceOperator(Operator):
    """Holds an fb_operator handle; shared apply plumbing."""

    graph_safe = True  # apply_into = device launches only (capturable in a CUDA graph)
    handle = None
    in_size = 0
    out_size = 0

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None and _lib.lib is not None:
            _lib.lib.fb_operator_destroy(h)
            self.handle = None

    @property
    def fast_path(self):
        return bool(_lib.lib.fb_operator_fast_path(self.handle))

    @property
    def device_bytes(self):
        return int(_lib.lib.fb_operator_device_bytes(self.handle))

    def _check_in(self, x):
        if tuple(x.shape) != (self.in_size,):
            raise ValueError(f"operand has shape {tuple(x.shape)}, expected ({self.in_size},)")

    def apply_into(self, x, y, stream=None):
        """y = A x on device tensors (no allocation, no synchronisation)."""
        _lib.check(_lib.lib.fb_operator_apply(self.handle, x.data_ptr(), y.data_ptr(),
                                              dev.stream_handle() if stream is None else stream))
        return y

    def apply(self, x):
        self._check_in(x)
        xd, host = dev.DeviceIn.get(x)
        y = dev.empty(self.out_size)
        self.apply_into(xd, y)
        return dev.to_host(y) if host else y

    def _create(self, kind, rv, rp, vdim, points, B, D, Bp, Dp, wdet, stiff, grad, geom,
                c=0.0, nu=1.0):
        h = C.c_void_p()
        pts = np.ascontiguousarray(points, dtype=np.float64)
        if _is_device_geom(geom):
            corners = np.ascontiguousarray(geom.mesh.corners, dtype=np.float64)
            w1 = np.ascontiguousarray(geom.rule.weights, dtype=np.float64)
            _lib.check(_lib.lib.fb_operator_create_geom(
                _lib.KIND[kind], rv.handle, rp.handle if rp else None, vdim, len(pts),
                _lib.ptr(pts), _lib.ptr(w1), _lib.ptr(B), _lib.ptr(D), _lib.ptr(Bp), _lib.ptr(Dp),
                _lib.ptr(corners), float(c), float(nu), C.byref(h)))
        else:
            wdet = _lib.host_f64(wdet)
            stiff = _lib.host_f64(stiff)
            grad = _lib.host_f64(grad)
            _lib.check(_lib.lib.fb_operator_create(
                _lib.KIND[kind], rv.handle, rp.handle if rp else None, vdim, len(pts),
                _lib.ptr(pts), _lib.ptr(B), _lib.ptr(D), _lib.ptr(Bp), _lib.ptr(Dp),
                _lib.ptr(wdet), _lib.ptr(stiff), _lib.ptr(grad), C.byref(h)))
        self.handle = h

    def device_factors(self):
        """Element-blocked (ne, K, nq^d) factors read back from the device."""
        n = int(_lib.lib.fb_operator_factor_count(self.handle))
        out = np.empty(n)
        _lib.check(_lib.lib.fb_operator_factors(self.handle, _lib.ptr(out), n))
        return out


class _SquareOperator(_DeviceOperator):
    kind = None

    def __init__(self, space, geom):
        _check_rule_match(space, geom)
        t0 = time.perf_counter()
        self.space = space
        self.geom = geom
        self.factors = QPointFactors()
        self.rule_points = np.asarray(geom.rule.points, dtype=np.float64)
        self.B, self.D = _eval_matrices(space, self.rule_points)
        self.restriction = restriction(space)
        if not _is_device_geom(geom):
            self._build_factors()
        self._create(self.kind, self.restriction, None, space.vdim, self.rule_points, self.B,
                     self.D, None, None, self.factors.wdet, self.factors.stiff, None, geom,
                     c=getattr(self, "c", 0.0), nu=getattr(self, "nu", 1.0))
        self.setup_seconds = time.perf_counter() - t0
        n = space.ndofs
        self.shape = (n, n)
        self.in_size = self.out_size = n

    def _build_factors(self):
        raise NotImplementedError


class MassOperator(_SquareOperator):
    kind = "mass"

    def _build_factors(self):
        self.factors.wdet = _mass_factor(self.geom)


class StiffnessOperator(_SquareOperator):
    kind = "stiffness"

    def __init__(self, space, geom, nu=1.0):
        self.nu = float(nu)
        super().__init__(space, geom)

    def _build_factors(self):
        self.factors.stiff = _stiffness_factor(self.geom, self.nu)


class HelmholtzOperator(_SquareOperator):
    """c * mass + stiffness in one fused sweep."""

    kind = "helmholtz"

    def __init__(self, space, geom, c, nu=1.0):
        self.c = float(c)
        self.nu = float(nu)
        super().__init__(space, geom)

    def _build_factors(self):
        self.factors.wdet = self.c * _mass_factor(self.geom)
        self.factors.stiff = _stiffness_factor(self.geom, self.nu)


class _MixedOperator(_DeviceOperator):
    kind = None
    _msg = ""

    def __init__(self, vspace, pspace, geom):
        _check_rule_match(vspace, geom)
        if vspace.vdim != vspace.dim or pspace.vdim != 1:
            raise ValueError(self._msg)
        t0 = time.perf_counter()
        self.vspace = vspace
        self.pspace = pspace
        self.geom = geom
        pts = np.asarray(geom.rule.points, dtype=np.float64)
        self.rule_points = pts
        self.Bv, self.Dv = _eval_matrices(vspace, pts)
        self.Bp, self.Dp = _eval_matrices(pspace, pts)
        self.factors = QPointFactors(grad=None if _is_device_geom(geom) else _grad_factor(geom))
        self.rv = restriction(vspace)
        self.rp = restriction(pspace)
        self._create(self.kind, self.rv, self.rp, vspace.dim, pts, self.Bv, self.Dv, self.Bp,
                     self.Dp, None, None, self.factors.grad, geom)
        self.setup_seconds = time.perf_counter() - t0


class GradientOperator(_MixedOperator):
    """Weak gradient (G q)_i = int phi_i . grad q (mfop.py:247-288)."""

    kind = "gradient"
    _msg = "gradient expects a vector velocity space and scalar pressure space"

    def __init__(self, vspace, pspace, geom):
        super().__init__(vspace, pspace, geom)
        self.shape = (vspace.ndofs, pspace.ndofs_scalar)
        self.in_size, self.out_size = pspace.ndofs_scalar, vspace.ndofs

    def apply_transpose_into(self, v, out, stream=None):
        _lib.check(_lib.lib.fb_operator_apply_transpose(
            self.handle, v.data_ptr(), out.data_ptr(),
            dev.stream_handle() if stream is None else stream))
        return out

    def apply_transpose(self, v):
        if tuple(v.shape) != (self.out_size,):
            raise ValueError(f"operand has shape {tuple(v.shape)}, expected ({self.out_size},)")
        vd, host = dev.DeviceIn.get(v)
        out = dev.empty(self.in_size)
        self.apply_transpose_into(vd, out)
        return dev.to_host(out) if host else out


class DivergenceOperator(_MixedOperator):
    """Weak divergence (D u)_i = int psi_i div u (mfop.py:291-319)."""

    kind = "divergence"
    _msg = "divergence expects a vector velocity space and scalar pressure space"

    def __init__(self, vspace, pspace, geom):
        super().__init__(vspace, pspace, geom)
        self.shape = (pspace.ndofs_scalar, vspace.ndofs)
        self.in_size, self.out_size = vspace.ndofs, pspace.ndofs_scalar


class ConvectionOperator(_DeviceOperator):
    """Nonlinear convection load N(u)_i = int ((u . grad) u) . phi_i
    (mfop.py:322-358), used by the projection stepper's extrapolated
    convection term (timeint.py:356).  One kernel computes the values of all
    components and the physical gradient of the output component at the
    quadrature points (factors wdet Jinv, the gradient set) and the
    transposed interpolation; the E->L sum is the deterministic one."""

    kind = "convection"

    def __init__(self, vspace, geom):
        _check_rule_match(vspace, geom)
        if vspace.vdim != vspace.dim:
            raise ValueError("convection expects a vector space with vdim == dim")
        t0 = time.perf_counter()
        self.vspace = vspace
        self.geom = geom
        pts = np.asarray(geom.rule.points, dtype=np.float64)
        self.rule_points = pts
        self.B, self.D = _eval_matrices(vspace, pts)
        self.factors = QPointFactors(grad=None if _is_device_geom(geom) else _grad_factor(geom))
        self.restriction = restriction(vspace)
        self._create(self.kind, self.restriction, None, vspace.dim, pts, self.B, self.D, None,
                     None, None, None, self.factors.grad, geom)
        n = vspace.ndofs
        self.shape = (n, n)
        self.in_size = self.out_size = n
        self.setup_seconds = time.perf_counter() - t0


def _curl_factor(geom, nu):
    """(ne, nq, 1 + d^2): nu * wdet, then Jinv[m][k] (m-major)."""
    wdet = _mass_factor(geom)
    d = geom.jinv.shape[-1]
    out = np.empty(wdet.shape + (1 + d * d,))
    out[..., 0] = nu * wdet
    out[..., 1:] = geom.jinv.reshape(wdet.shape + (d * d,))
    return out


class CurlCurlOperator(_DeviceOperator):
    """Weak rotational viscous term int nu (curl u) . (curl v) (mfop.py:361-413).
    One kernel computes the physical gradients of every velocity component,
    the weighted vorticity and the transposed gradient of the output
    component; deterministic E->L sum."""

    kind = "curlcurl"

    def __init__(self, vspace, geom, nu=1.0):
        _check_rule_match(vspace, geom)
        if vspace.vdim != vspace.dim:
            raise ValueError("curl-curl expects a vector space with vdim == dim")
        t0 = time.perf_counter()
        self.vspace = vspace
        self.geom = geom
        self.nu = float(nu)
        pts = np.asarray(geom.rule.points, dtype=np.float64)
        self.rule_points = pts
        self.B, self.D = _eval_matrices(vspace, pts)
        self.factors = QPointFactors()
        curl = None if _is_device_geom(geom) else _curl_factor(geom, self.nu)
        self.restriction = restriction(vspace)
        self._create(self.kind, self.restriction, None, vspace.dim, pts, self.B, self.D, None,
                     None, None, None, curl, geom, nu=self.nu)
        n = vspace.ndofs
        self.shape = (n, n)
        self.in_size = self.out_size = n
        self.setup_seconds = time.perf_counter() - t0


class ConstrainedOperator(Operator):
    """Identity on constrained rows, the inner operator elsewhere
    (mfop.py:416-433): xi = x; xi[C] = 0; y = A xi; y[C] = x[C]."""

    def __init__(self, op, constrained_dofs):
        self.op = op
        self.constrained = np.asarray(constrained_dofs, dtype=np.int64)
        self.shape = op.shape
        self._dofs_dev = None
        self._work = None

    @property
    def graph_safe(self):
        return bool(getattr(self.op, "graph_safe", False)) and hasattr(self.op, "apply_into")

    def _dofs(self):
        if self._dofs_dev is None:
            self._dofs_dev = torch.from_numpy(self.constrained).to(dev.device())
        return self._dofs_dev

    def apply_into(self, x, y, stream=None):
        st = dev.stream_handle() if stream is None else stream
        n = x.shape[0]
        if self._work is None or self._work.shape[0] != n:
            self._work = dev.empty(n)
        d = self._dofs()
        _lib.check(_lib.lib.fb_mask_copy_zero(x.data_ptr(), self._work.data_ptr(), n,
                                              d.data_ptr(), d.shape[0], st))
        if hasattr(self.op, "apply_into"):
            self.op.apply_into(self._work, y, stream)
        else:
            y.copy_(dev.to_device(self.op.apply(self._work)))
        _lib.check(_lib.lib.fb_mask_restore(x.data_ptr(), y.data_ptr(), d.data_ptr(), d.shape[0],
                                            st))
        return y

    def apply(self, x):
        xd, host = dev.DeviceIn.get(x)
        y = dev.empty(self.shape[0])
        self.apply_into(xd, y)
        return dev.to_host(y) if host else y


def setup(kind, space=None, geom=None, vspace=None, pspace=None, nu=1.0, c=0.0):
    """Factory over the supported kinds (mfop.py:436-452)."""
    if kind == "mass":
        return MassOperator(space, geom)
    if kind == "stiffness":
        return StiffnessOperator(space, geom, nu=nu)
    if kind == "helmholtz":
        return HelmholtzOperator(space, geom, c, nu=nu)
    if kind == "gradient":
        return GradientOperator(vspace, pspace, geom)
    if kind == "divergence":
        return DivergenceOperator(vspace, pspace, geom)
    if kind == "convection":
        return ConvectionOperator(vspace or space, geom)
    if kind == "curlcurl":
        return CurlCurlOperator(vspace or space, geom, nu=nu)
    raise ValueError(f"unknown operator kind {kind!r}")


# -- right-hand-side formation (host setup; outside the hot path) --------------

def _tensor_t(fq, Bt, d):
    """(ne, nq^d) -> (ne, n^d): B^T applied along every axis."""
    ne, q = fq.shape[0], Bt.shape[1]
    t = fq.reshape((ne,) + (q,) * d)
    if d == 2:
        t = np.einsum("ai,eji->eja", Bt, t)
        t = np.einsum("bj,eja->eba", Bt, t)
    else:
        t = np.einsum("ai,ekji->ekja", Bt, t)
        t = np.einsum("bj,ekja->ekba", Bt, t)
        t = np.einsum("ck,ekba->ecba", Bt, t)
    return t.reshape(ne, -1)


def load_vector(space, geom, f):
    """Weak forcing b_i = (f, phi_i) with f sampled at the quadrature points
    (the reference's load_vector, mfop.py:600-620)."""
    _check_rule_match(space, geom)
    B, _ = _eval_matrices(space, np.asarray(geom.rule.points))
    wdet = geom.detj * geom.w[None, :]
    xq = geom.xq.reshape(-1, space.dim)
    vals = np.asarray(f(xq), dtype=np.float64)
    if vals.ndim == 1:
        vals = vals[:, None]
    if vals.shape != (xq.shape[0], space.vdim):
        raise ValueError(f"forcing returned shape {vals.shape}, expected ({xq.shape[0]}, {space.vdim})")
    ne, nq = geom.detj.shape
    ns = space.ndofs_scalar
    out = np.empty(space.ndofs)
    for c in range(space.vdim):
        loc = _tensor_t(vals[:, c].reshape(ne, nq) * wdet, B.T, space.dim)
        out[c * ns:(c + 1) * ns] = np.bincount(space.element_dofs.ravel(), weights=loc.ravel(),
                                                minlength=ns)
    return out


def boundary_normal_flux(space, g, attributes=None, n_quad=None):
    """Boundary load b_i = int_faces psi_i (g . n) (mfop.py:623-684): a device
    SpMV of a face matrix built once per space (boundary.py)."""
    from . import boundary
    return boundary.boundary_normal_flux(space, g, attributes=attributes, n_quad=n_quad)


def boundary_rotational_rhs(vspace, pspace, u, nu=1.0, attributes=None, n_quad=None):
    """Pressure load r_j = -nu int_faces (n x curl u) . grad psi_j
    (mfop.py:687-807): a device SpMV of a face matrix built once per space
    pair (boundary.py).  Device u gives a device result, host u a host one."""
    from . import boundary
    return boundary.boundary_rotational_rhs(vspace, pspace, u, nu=nu, attributes=attributes,
                                            n_quad=n_quad)
