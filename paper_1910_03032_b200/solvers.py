"""Krylov solvers and LOR preconditioners on the B200: drop-in for `solvers`.

Same API as the reference (solvers.py:25-425): ``SolverConfig``,
``SolveReport``, ``cg``, ``fgmres``, ``DiagonalPreconditioner``,
``collocated_mass_diagonal``, ``deflate_mean``, ``MeanProjector``,
``ILU0Smoother``, ``LORPreconditioner``, ``BlockDiagonalPreconditioner``,
``InnerCG``.  The iterations keep the reference recurrences exactly
(preconditioned-residual stopping test, true residual every 50 CG steps,
right-preconditioned flexible GMRES with modified Gram-Schmidt, restart 50)
but every vector lives on the device: dots, updates, SpMVs, triangular
solves and operator applies are CUDA kernels of libfbb200, scalars such as
alpha stay on the device, and the host reads back a few scalars per
iteration for the stopping test.  A numpy right-hand side gives a numpy
solution (drop-in); a CUDA tensor gives a CUDA tensor.

Objects exposing ``apply_into(x, y)`` (this package's operators and
preconditioners) run fully on the device.  scipy sparse matrices are moved
to the device once.  Any other ``.apply``/callable is treated as a host
(numpy) function and called through a device<->host round trip.
"""

import gc
import math
import os
import threading
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse as sp
import scipy.sparse.linalg as spla
import torch

from . import _lib
from . import device as dev
from . import lor as lor_mod
from . import vec
from .geometry import compute_geometric_factors
from .quadrature import GAUSS_LOBATTO, quadrature_rule
from .spaces import FESpace


@dataclass
class SolverConfig:
    rel_tol: float = 1e-8
    abs_tol: float = 0.0
    max_iters: int = 500
    restart: int = 50
    label: str = ""


@dataclass
class SolveReport:
    converged: bool
    iterations: int
    final_relres: float
    seconds: float
    label: str = ""
    residuals: list = field(default_factory=list)

    def __str__(self):
        tag = "converged" if self.converged else "NOT converged"
        name = f"{self.label}: " if self.label else ""
        return (f"{name}{tag} in {self.iterations} iterations, "
                f"relres {self.final_relres:.3e}, {self.seconds:.3f}s")


# Smoother used by LORPreconditioner when none is given: "block" (device
# block-Jacobi ILU(0), the B200 path) or "global" (the reference's ILU(0)).
DEFAULT_SMOOTHER = "block"


# -- operand normalisation ------------------------------------------------------

def _device_apply(A):
    """Return f(x, y) computing y = A x on device tensors."""
    if hasattr(A, "apply_into"):
        return A.apply_into
    if sp.issparse(A):
        D = vec.DeviceCSR(A)
        return D.apply_into
    fn = A.apply if hasattr(A, "apply") else A
    if not callable(fn):
        raise TypeError(f"cannot interpret {type(A)} as an operator")

    def host_apply(x, y):
        y.copy_(dev.to_device(np.asarray(fn(dev.to_host(x)), dtype=np.float64)))
        return y

    return host_apply


def _device_project(project):
    if hasattr(project, "apply_into"):
        return project.apply_into

    def host_project(x, y):
        y.copy_(dev.to_device(np.asarray(project(dev.to_host(x)), dtype=np.float64)))
        return y

    return host_project


def _as_apply(A):
    """Reference-compatible helper (solvers.py:50-57)."""
    if hasattr(A, "apply"):
        return A.apply
    if sp.issparse(A):
        return lambda v: A @ v
    if callable(A):
        return A
    raise TypeError(f"cannot interpret {type(A)} as an operator")


class _DeviceMixin:
    """numpy-or-tensor `apply` on top of a device `apply_into`."""

    def apply(self, r):
        rd, host = dev.DeviceIn.get(r)
        out = torch.empty_like(rd)
        self.apply_into(rd, out)
        return dev.to_host(out) if host else out

    def __call__(self, r):
        return self.apply(r)


# -- mean deflation ---------------------------------------------------------------

class MeanProjector(_DeviceMixin):
    """v - (sum w_i v_i / sum w_i) 1, or v - mean(v) (solvers.py:60-74)."""

    def __init__(self, weights=None):
        self.weights = weights
        self._w = None
        self._den = None

    def apply_into(self, v, out, stream=None):
        n = v.shape[0]
        if self._w is None or self._w.shape[0] != n:
            if self.weights is None:
                self._w = torch.ones(n, dtype=torch.float64, device=dev.device())
                self._den = float(n)
            else:
                w = np.asarray(self.weights, dtype=np.float64)
                self._w = dev.to_device(w)
                self._den = float(w.sum())
        num = vec.workspace(n).scalars[15:16]
        vec.dot_into(self._w, v, num, stream)
        vec.shift_ratio(v, num, self._den, out, stream)
        return out


class _StreamMeanProjector(MeanProjector):
    """MeanProjector with private reduction scratch (no shared vec.workspace
    slot), for preconditioner clones running on concurrent streams."""

    def apply_into(self, v, out, stream=None):
        n = v.shape[0]
        if self._w is None or self._w.shape[0] != n:
            self._w = torch.ones(n, dtype=torch.float64, device=dev.device())
            self._den = float(n)
            self._num = dev.zeros(1)
            self._part = dev.zeros(int(_lib.lib.fb_dot_partials(n)))
        _lib.check(_lib.lib.fb_dot(n, self._w.data_ptr(), v.data_ptr(), self._part.data_ptr(),
                                   self._num.data_ptr(), vec._st(stream)))
        vec.shift_ratio(v, self._num, self._den, out, stream)
        return out


def deflate_mean(v, weights=None):
    return MeanProjector(weights).apply(v)


class DiagonalPreconditioner(_DeviceMixin):
    graph_safe = True

    def __init__(self, diag):
        self.inv = 1.0 / np.asarray(diag, dtype=np.float64)
        self._inv = None

    def apply_into(self, r, z, stream=None):
        if self._inv is None:
            self._inv = dev.to_device(self.inv)
        return vec.vmul(self._inv, r, z, stream)


def collocated_mass_diagonal(space, constrained=None):
    """GLL-collocated (lumped) mass diagonal w_i det J(x_i) (solvers.py:87-105)."""
    rule = quadrature_rule(GAUSS_LOBATTO, space.p + 1)
    geom = compute_geometric_factors(space.mesh, rule)
    vals = geom.detj * geom.w[None, :]
    diag = np.bincount(space.element_dofs.ravel(), weights=vals.ravel(),
                       minlength=space.ndofs_scalar)
    if space.vdim > 1:
        diag = np.tile(diag, space.vdim)
    if constrained is not None and len(constrained):
        diag = diag.copy()
        diag[np.asarray(constrained, dtype=np.int64)] = 1.0
    return diag


# -- Krylov --------------------------------------------------------------------------

# device-resident PCG (CUDA graph with a conditional WHILE node, fb_graph.cu)
# for single-GPU device operators up to this size; FB_CG_GRAPH=0 disables it
GRAPH_MAX_N = 20_000_000
TRUE_RESIDUAL_PERIOD = 50  # solvers.py:145-150



_gc_lock = threading.Lock()
_gc_state = {"depth": 0, "was_enabled": False}


def _gc_pause(enter):
    """Cyclic GC off while any thread captures a CUDA graph (in-process ranks
    capture concurrently): a collected object's __del__ may cudaFree, which
    invalidates a capture in progress."""
    with _gc_lock:
        if enter:
            if _gc_state["depth"] == 0:
                _gc_state["was_enabled"] = gc.isenabled()
                gc.disable()
            _gc_state["depth"] += 1
        else:
            _gc_state["depth"] -= 1
            if _gc_state["depth"] == 0 and _gc_state["was_enabled"]:
                gc.enable()


class _CGGraph:
    """One captured PCG iteration for a fixed (A, precond, n): the body of a
    device-side while loop.  Vectors, scalars and dot partials are owned
    here, so the graph's pointers stay valid for every solve."""

    def __init__(self, A, precond, n, cap):
        self.A, self.precond, self.n, self.cap = A, precond, n, cap
        self.apply_A = _device_apply(A)
        self.M = _device_apply(precond) if precond is not None else None
        self.x, self.r, self.z, self.p, self.Ap, self.tmp, self.b = (dev.empty(n) for _ in range(7))
        self.s = dev.zeros(8)  # rz, pAp, alpha, rz_new, beta
        self.cfgd = dev.zeros(2)  # norm0, rel_tol
        self.state = torch.zeros(4, dtype=torch.int32, device=dev.device())
        self.hist = dev.zeros(cap + 2)
        npart = int(_lib.lib.fb_dot_partials(n))
        self.part = [dev.empty(npart), dev.empty(npart)]
        self.stream = torch.cuda.Stream()
        self.graph = None

    def __del__(self):
        g = getattr(self, "graph", None)
        if g and _lib is not None and _lib.lib is not None:
            _lib.lib.fb_while_graph_destroy(g)

    def _dot(self, x, y, k, slot, st):
        _lib.check(_lib.lib.fb_dot(self.n, x.data_ptr(), y.data_ptr(), self.part[k].data_ptr(),
                                   self.s[slot:slot + 1].data_ptr(), st))

    def _iteration(self, st, true_res, handle, in_graph):
        n = self.n
        self.apply_A(self.p, self.Ap)
        self._dot(self.p, self.Ap, 0, 1, st)
        s = self.s
        _lib.check(_lib.lib.fb_cg_update(n, s[0:1].data_ptr(), s[1:2].data_ptr(),
                                         s[2:3].data_ptr(), self.p.data_ptr(), self.Ap.data_ptr(),
                                         self.x.data_ptr(), self.r.data_ptr(),
                                         0 if true_res else 1, st))
        if true_res:
            self.apply_A(self.x, self.tmp)
            vec.copy(self.b, self.r, st)
            vec.axpby(-1.0, self.tmp, 1.0, self.r, st)
        if self.M is not None:
            self.M(self.r, self.z)
        else:
            vec.copy(self.r, self.z, st)
        self._dot(self.r, self.z, 1, 3, st)
        _lib.check(_lib.lib.fb_cg_check(handle, in_graph, s.data_ptr(), self.state.data_ptr(),
                                        self.hist.data_ptr(), self.cfgd.data_ptr(),
                                        TRUE_RESIDUAL_PERIOD, st))
        _lib.check(_lib.lib.fb_xpby_dev(n, self.z.data_ptr(), s[4:5].data_ptr(),
                                        self.p.data_ptr(), st))

    def _capture(self, st):
        import ctypes as C
        g = C.c_void_p()
        _lib.check(_lib.lib.fb_while_graph_create(C.byref(g)))
        self.graph = g
        handle = _lib.lib.fb_while_graph_handle(g)
        # no cyclic GC while capturing: a collected space / transfer / matrix
        # frees device memory in its __del__, and a cudaFree inside the capture
        # invalidates it (seen as an order-dependent "previous error during
        # capture" once earlier tests left such cycles behind)
        _gc_pause(True)
        _lib.check(_lib.lib.fb_while_graph_begin(g, st))
        try:
            self._iteration(st, False, handle, 1)
        finally:
            try:
                _lib.check(_lib.lib.fb_while_graph_end(g, st))
            finally:
                _gc_pause(False)

    def solve(self, bd, cfg, t0):
        cur = torch.cuda.current_stream()
        self.stream.wait_stream(cur)
        with torch.cuda.stream(self.stream):
            st = self.stream.cuda_stream
            vec.copy(bd, self.b, st)
            vec.copy(self.b, self.r, st)  # A(0) == 0 exactly
            self.x.zero_()
            if self.M is not None:
                self.M(self.r, self.z)
            else:
                vec.copy(self.r, self.z, st)
            self._dot(self.r, self.z, 1, 0, st)
            rz = float(self.s[0].item())
            norm0 = math.sqrt(abs(rz))
            history = [1.0]
            if norm0 == 0.0 or norm0 <= cfg.abs_tol:
                cur.wait_stream(self.stream)
                return self.x.clone(), SolveReport(True, 0, 0.0, time.perf_counter() - t0,
                                                   cfg.label, history)
            vec.copy(self.z, self.p, st)
            self.cfgd.copy_(torch.tensor([norm0, cfg.rel_tol], dtype=torch.float64))
            self.state.copy_(torch.tensor([0, 0, cfg.max_iters, 0], dtype=torch.int32))
            if self.graph is None:
                self.apply_A(self.p, self.Ap)  # lazy workspaces are allocated before capture
                self._capture(st)
            it, stop = 0, 0
            while True:
                if (it + 1) % TRUE_RESIDUAL_PERIOD == 0:
                    self._iteration(st, True, 0, 0)
                else:
                    _lib.check(_lib.lib.fb_while_graph_launch(self.graph, st))
                it, stop = (int(v) for v in self.state[:2].tolist())
                if stop or it >= cfg.max_iters:
                    break
            hist = self.hist[:it + 1].tolist()
            x = self.x.clone()
        cur.wait_stream(self.stream)
        history = [1.0] + hist[1:it + 1] if stop != 2 else [1.0] + hist[1:it]
        relres = history[-1]
        converged = stop == 1 or cfg.rel_tol == 0.0
        return x, SolveReport(converged, it, relres, time.perf_counter() - t0, cfg.label, history)


def _cg_graph_for(A, precond, n, cap):
    cache = A.__dict__.setdefault("_fb_cg_graphs", {})
    key = (id(precond), n)
    g = cache.get(key)
    if g is None or g.precond is not precond or g.cap < cap:
        g = _CGGraph(A, precond, n, max(cap, 512))
        cache[key] = g
    return g


def _graph_eligible(A, precond, x0, project, inner, n):
    return (inner is None and project is None and x0 is None and n <= GRAPH_MAX_N
            and bool(getattr(A, "graph_safe", False)) and hasattr(A, "apply_into")
            and (precond is None or bool(getattr(precond, "graph_safe", False)))
            and os.environ.get("FB_CG_GRAPH", "1") != "0")


def cg(A, b, precond=None, config=None, x0=None, project=None, inner=None):
    """Preconditioned CG with the reference recurrence (solvers.py:108-169).
    inner(x, y, out): the inner product into a 1-element device tensor
    (default: the deterministic libfbb200 dot; the sharded solver passes an
    owned-slice dot + all-reduce).  Single-GPU device operators run the
    whole loop on the device (_CGGraph): same kernels, same arithmetic,
    no per-iteration host synchronisation."""
    cfg0 = config or SolverConfig()
    bd0, host0 = dev.DeviceIn.get(b)
    if _graph_eligible(A, precond, x0, project, inner, bd0.shape[0]):
        t0 = time.perf_counter()
        x, rep = _cg_graph_for(A, precond, bd0.shape[0], cfg0.max_iters).solve(bd0, cfg0, t0)
        return (dev.to_host(x) if host0 else x), rep
    dot_into = inner if inner is not None else vec.dot_into
    apply_A = _device_apply(A)
    M = _device_apply(precond) if precond is not None else None
    proj = _device_project(project) if project is not None else None
    cfg = config or SolverConfig()
    t0 = time.perf_counter()
    bd, host = dev.DeviceIn.get(b)
    n = bd.shape[0]
    x = dev.zeros(n) if x0 is None else dev.to_device(x0).clone()
    r = dev.empty(n)
    tmp = dev.empty(n)
    z = dev.empty(n)
    # device scalars: 0 rz, 1 pAp, 2 alpha, 3 rz_new
    s = dev.zeros(4)
    if x0 is None:
        vec.copy(bd, r)  # A(0) == 0 exactly
    else:
        apply_A(x, tmp)
        vec.copy(bd, r)
        vec.axpby(-1.0, tmp, 1.0, r)
    if proj is not None:
        proj(r, r)
    if M is not None:
        M(r, z)
    else:
        vec.copy(r, z)
    if proj is not None:
        proj(z, z)
    dot_into(r, z, s[0:1])
    rz = float(s[0].item())
    norm0 = math.sqrt(abs(rz))
    history = [1.0]

    def done(conv, its, rel):
        return (dev.to_host(x) if host else x), SolveReport(conv, its, rel,
                                                           time.perf_counter() - t0, cfg.label,
                                                           history)

    if norm0 == 0.0 or norm0 <= cfg.abs_tol:
        return done(True, 0, 0.0)
    p = z.clone()
    Ap = dev.empty(n)
    relres = 1.0
    it = 0
    converged = False
    old, new = 0, 3  # device slots of rz and rz_new, swapped every iteration (no copy)
    for it in range(1, cfg.max_iters + 1):
        apply_A(p, Ap)
        dot_into(p, Ap, s[1:2])
        # fused: alpha = rz / pAp (0 if pAp <= 0); x += alpha p; r -= alpha Ap
        true_res = it % 50 == 0
        vec.cg_update(s[old:old + 1], s[1:2], s[2:3], p, Ap, x, r, update_r=not true_res)
        if true_res:
            apply_A(x, tmp)
            vec.copy(bd, r)
            vec.axpby(-1.0, tmp, 1.0, r)
            if proj is not None:
                proj(r, r)
        if M is not None:
            M(r, z)
        else:
            vec.copy(r, z)
        if proj is not None:
            proj(z, z)
        dot_into(r, z, s[new:new + 1])
        vals = s.tolist()
        pAp, rz_new = vals[1], vals[new]
        if pAp <= 0.0:
            break
        relres = math.sqrt(abs(rz_new)) / norm0
        history.append(relres)
        if cfg.rel_tol > 0.0 and relres <= cfg.rel_tol:
            converged = True
            break
        if rz_new == 0.0:
            converged = True
            break
        vec.xpby_ratio(z, s[new:new + 1], s[old:old + 1], p)  # p = z + (rz_new / rz) p
        old, new = new, old
    if cfg.rel_tol == 0.0:
        converged = True
    return done(converged, it, relres)


def minres(A, b, precond=None, config=None, x0=None, shift=0.0):
    """Preconditioned MINRES for symmetric (indefinite) A with an SPD
    preconditioner -- the Krylov method the north star names for the
    block-diagonal-preconditioned Stokes problem.  The
    reference has no MINRES; this restates the Paige-Saunders recurrence and
    stopping tests of scipy.sparse.linalg.minres (the oracle of
    tests/test_gpu_minres.py) with device vectors and libfbb200 kernels: per
    iteration one A apply, one preconditioner apply, three inner products
    (the only host round trips) and six axpy-type updates.
    Returns (x, SolveReport); converged means scipy's istop in {1, 2}."""
    apply_A = _device_apply(A)
    M = _device_apply(precond) if precond is not None else None
    cfg = config or SolverConfig()
    rtol, maxiter = cfg.rel_tol, cfg.max_iters
    eps = float(np.finfo(np.float64).eps)
    t0 = time.perf_counter()
    bd, host = dev.DeviceIn.get(b)
    n = bd.shape[0]
    sc = dev.empty(1)

    def dot(u, v):
        vec.dot_into(u, v, sc)
        return float(sc.item())

    x = dev.zeros(n) if x0 is None else dev.to_device(x0).clone()
    R1 = dev.empty(n)
    if x0 is None:
        vec.copy(bd, R1)
    else:
        apply_A(x, R1)
        vec.axpby(1.0, bd, -1.0, R1)
    Y = dev.empty(n)
    if M is not None:
        M(R1, Y)
    else:
        vec.copy(R1, Y)
    beta1 = dot(R1, Y)

    def done(conv, its, rel, hist):
        return (dev.to_host(x) if host else x), SolveReport(conv, its, rel,
                                                           time.perf_counter() - t0, cfg.label,
                                                           hist)

    if beta1 < 0:
        raise ValueError("indefinite preconditioner")
    if beta1 == 0 or dot(bd, bd) == 0:
        return done(True, 0, 0.0, [0.0])
    beta1 = math.sqrt(beta1)
    R2 = R1.clone()
    T, V = dev.empty(n), dev.empty(n)
    W, W1, W2 = dev.zeros(n), dev.zeros(n), dev.zeros(n)
    oldb, beta, dbar, epsln, phibar = 0.0, beta1, 0.0, 0.0, beta1
    rhs1, rhs2, tnorm2, gmax, gmin = beta1, 0.0, 0.0, 0.0, float(np.finfo(np.float64).max)
    cs, sn = -1.0, 0.0
    istop, itn, rnorm = 0, 0, beta1
    history = [1.0]
    while itn < maxiter:
        itn += 1
        vec.scale(1.0 / beta, Y, V)            # v = y / beta
        apply_A(V, T)                           # y = A v - shift v
        if shift:
            vec.axpby(-shift, V, 1.0, T)
        if itn >= 2:
            vec.axpby(-beta / oldb, R1, 1.0, T)
        alfa = dot(V, T)
        vec.axpby(-alfa / beta, R2, 1.0, T)
        R1, R2, T = R2, T, R1                   # r1 <- r2, r2 <- y
        if M is not None:                       # y = M r2
            M(R2, Y)
        else:
            vec.copy(R2, Y)
        oldb = beta
        beta = dot(R2, Y)
        if beta < 0:
            raise ValueError("non-symmetric matrix")
        beta = math.sqrt(beta)
        tnorm2 += alfa ** 2 + oldb ** 2 + beta ** 2
        if itn == 1 and beta / beta1 <= 10 * eps:
            istop = -1
        oldeps = epsln
        delta = cs * dbar + sn * alfa
        gbar = sn * dbar - cs * alfa
        epsln = sn * beta
        dbar = -cs * beta
        root = math.hypot(gbar, dbar)
        gamma = max(math.hypot(gbar, beta), eps)
        cs, sn = gbar / gamma, beta / gamma
        phi = cs * phibar
        phibar = sn * phibar
        denom = 1.0 / gamma
        W1, W2, W = W2, W, W1                   # w1 <- w2, w2 <- w
        vec.scale(denom, V, W)                  # w = (v - oldeps w1 - delta w2) / gamma
        vec.axpby(-oldeps * denom, W1, 1.0, W)
        vec.axpby(-delta * denom, W2, 1.0, W)
        vec.axpby(phi, W, 1.0, x)
        gmax, gmin = max(gmax, gamma), min(gmin, gamma)
        z = rhs1 / gamma
        rhs1, rhs2 = rhs2 - delta * z, -epsln * z
        Anorm = math.sqrt(tnorm2)
        ynorm = math.sqrt(dot(x, x))
        epsx = Anorm * ynorm * eps
        rnorm = phibar
        test1 = math.inf if (ynorm == 0 or Anorm == 0) else rnorm / (Anorm * ynorm)
        test2 = math.inf if Anorm == 0 else root / Anorm
        history.append(rnorm / beta1)
        if istop == 0:
            if 1 + test2 <= 1:
                istop = 2
            if 1 + test1 <= 1:
                istop = 1
            if itn >= maxiter:
                istop = 6
            if gmax / gmin >= 0.1 / eps:
                istop = 4
            if epsx >= beta1:
                istop = 3
            if test2 <= rtol:
                istop = 2
            if test1 <= rtol:
                istop = 1
        if istop != 0:
            break
    return done(istop in (1, 2), itn, rnorm / beta1, history)


def fgmres(A, b, precond=None, config=None, x0=None, project=None):
    """Right-preconditioned flexible GMRES(m) with MGS (solvers.py:172-254)."""
    apply_A = _device_apply(A)
    M = _device_apply(precond) if precond is not None else None
    proj = _device_project(project) if project is not None else None
    cfg = config or SolverConfig()
    t0 = time.perf_counter()
    bd, host = dev.DeviceIn.get(b)
    n = bd.shape[0]
    x = dev.zeros(n) if x0 is None else dev.to_device(x0).clone()
    r = dev.empty(n)
    tmp = dev.empty(n)

    def residual():
        apply_A(x, tmp)
        vec.copy(bd, r)
        vec.axpby(-1.0, tmp, 1.0, r)

    def norm(v):
        return math.sqrt(vec.dot(v, v).item())

    if x0 is None:
        vec.copy(bd, r)
    else:
        residual()
    beta0 = norm(r)
    history = [1.0]
    if beta0 == 0.0 or beta0 <= cfg.abs_tol:
        return (dev.to_host(x) if host else x), SolveReport(True, 0, 0.0,
                                                           time.perf_counter() - t0, cfg.label,
                                                           history)
    target = cfg.rel_tol * beta0
    m = cfg.restart
    V = torch.zeros((m + 1, n), dtype=torch.float64, device=dev.device())
    Z = torch.zeros((m, n), dtype=torch.float64, device=dev.device())
    hcol = dev.zeros(m + 2)
    w = dev.empty(n)
    it = 0
    relres = 1.0
    converged = False
    while it < cfg.max_iters and not converged:
        beta = norm(r)
        if beta <= max(target, cfg.abs_tol):
            converged = True
            break
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        vec.div_scalar(r, beta, V[0])
        j = -1
        for j in range(m):
            if it >= cfg.max_iters:
                j -= 1
                break
            it += 1
            zj = Z[j]
            if M is not None:
                M(V[j], zj)
            else:
                vec.copy(V[j], zj)
            if proj is not None:
                proj(zj, zj)
            apply_A(zj, w)
            for i in range(j + 1):
                vec.dot_into(V[i], w, hcol[i:i + 1])
                vec.axpy_dev(hcol[i:i + 1], V[i], w, -1)
            vec.dot_into(w, w, hcol[j + 1:j + 2])
            col = hcol[:j + 2].tolist()
            H[:j + 1, j] = col[:j + 1]
            H[j + 1, j] = math.sqrt(col[j + 1])
            if H[j + 1, j] > 1e-300:
                vec.div_scalar(w, H[j + 1, j], V[j + 1])
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            denom = np.hypot(H[j, j], H[j + 1, j])
            if denom == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j], sn[j] = H[j, j] / denom, H[j + 1, j] / denom
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            relres = abs(g[j + 1]) / beta0
            history.append(relres)
            if relres * beta0 <= max(target, cfg.abs_tol):
                converged = True
                break
        k = j + 1
        if k > 0:
            y = scipy.linalg.solve_triangular(H[:k, :k], g[:k], lower=False)
            for i in range(k):
                vec.axpby(float(y[i]), Z[i], 1.0, x)
        residual()
        relres = norm(r) / beta0
        if relres * beta0 <= max(target, cfg.abs_tol):
            converged = True
    return (dev.to_host(x) if host else x), SolveReport(converged, it, relres,
                                                       time.perf_counter() - t0, cfg.label,
                                                       history)


# -- ILU(0) smoother -----------------------------------------------------------------

def _first_touch_ordering(space):
    return lor_mod.first_touch_ordering(space)


def _degree_ladder(p):
    return lor_mod.degree_ladder(p)


class ILU0Smoother:
    """ILU(0) in a fixed ordering; forward = (LU)^-1, backward = (LU)^-T
    (solvers.py:269-311).  The factorisation runs once on the host (C++,
    the reference's IKJ variant); the four triangular solves run on the
    device.  A degenerate pivot falls back to damped Jacobi 0.6/diag."""

    def __init__(self, A, order, backend=None):
        A = A.tocsr()
        n = A.shape[0]
        self.n = n
        self.order = np.asarray(order, dtype=np.int64)
        Ap = A[self.order][:, self.order].tocsr()
        Ap.sort_indices()
        data = Ap.data.astype(np.float64, copy=True)
        fail = vec.ilu0_factor_host(Ap.indptr, Ap.indices, data)
        self.jacobi = None
        self.fail_row = fail
        if fail >= 0:
            diag = A.diagonal().copy()
            diag[diag == 0.0] = 1.0
            self.jacobi = 0.6 / diag
            self._jac = dev.to_device(self.jacobi)
            return
        F = sp.csr_matrix((data, Ap.indices.copy(), Ap.indptr.copy()), shape=(n, n))
        L = sp.tril(F, k=-1, format="csr")
        U = sp.triu(F, k=0, format="csr")
        self.L_factor, self.U_factor = L, U
        self._L = vec.TriSolve(L, lower=True, unit_diag=True)
        self._U = vec.TriSolve(U, lower=False, unit_diag=False)
        self._Ut = vec.TriSolve(U.T.tocsr(), lower=True, unit_diag=False)
        self._Lt = vec.TriSolve(L.T.tocsr(), lower=False, unit_diag=True)
        self._perm = torch.from_numpy(self.order.astype(np.int32)).to(dev.device())
        self._a = dev.empty(n)
        self._b = dev.empty(n)

    def forward_into(self, r, out, stream=None):
        if self.jacobi is not None:
            return vec.vmul(self._jac, r, out, stream)
        vec.permute(self._perm, r, self._a, scatter=False, stream=stream)
        self._L.solve_into(self._a, self._b, stream)
        self._U.solve_into(self._b, self._a, stream)
        return vec.permute(self._perm, self._a, out, scatter=True, stream=stream)

    def backward_into(self, r, out, stream=None):
        if self.jacobi is not None:
            return vec.vmul(self._jac, r, out, stream)
        vec.permute(self._perm, r, self._a, scatter=False, stream=stream)
        self._Ut.solve_into(self._a, self._b, stream)
        self._Lt.solve_into(self._b, self._a, stream)
        return vec.permute(self._perm, self._a, out, scatter=True, stream=stream)

    def forward(self, r):
        rd, host = dev.DeviceIn.get(r)
        out = torch.empty_like(rd)
        self.forward_into(rd, out)
        return dev.to_host(out) if host else out

    def backward(self, r):
        rd, host = dev.DeviceIn.get(r)
        out = torch.empty_like(rd)
        self.backward_into(rd, out)
        return dev.to_host(out) if host else out


def infer_counts(mesh):
    """Structured cell counts of a tensor-product mesh numbered x-fastest
    (cartesian_mesh, mesh.py:110-121), or None."""
    counts = getattr(mesh, "counts", None)
    if counts:
        return tuple(counts)
    ne, d = mesh.num_elements, mesh.dim
    cen = mesh.corners.mean(axis=1)
    wrap = np.flatnonzero(np.diff(cen[:, 0]) < 0)
    nx = int(wrap[0]) + 1 if wrap.size else ne
    if d == 2:
        return (nx, ne // nx) if ne % nx == 0 else None
    rows = cen[::nx, 1]
    wrap = np.flatnonzero(np.diff(rows) < 0)
    ny = int(wrap[0]) + 1 if wrap.size else ne // nx
    if ne % (nx * ny):
        return None
    return (nx, ny, ne // (nx * ny))


def element_block_ids(mesh, block):
    """Element -> block id for element-cube blocks of block^d elements."""
    ne, d = mesh.num_elements, mesh.dim
    counts = infer_counts(mesh)
    e = np.arange(ne)
    if counts is None or int(np.prod(counts)) != ne:
        return e // block ** d
    idx = []
    for a in range(d):
        idx.append((e % counts[a]) // block)
        e = e // counts[a]
    nb = [-(-counts[a] // block) for a in range(d)]
    bid = idx[-1]
    for a in range(d - 2, -1, -1):
        bid = bid * nb[a] + idx[a]
    return bid


class BlockILU0Smoother:
    """Block-Jacobi ILU(0) over element-cube blocks (SURVEY 8(e') scale mode).

    Every DoF joins the block of its first-touch owner element; couplings
    between blocks are dropped; inside a block the reference's first-touch
    order is kept, so each block's factor is exactly the reference ILU(0)
    restricted to that block.  Measured against the reference's global ILU:
    +0/+1 CG iterations (SURVEY 8(e')).  One kernel launch per sweep."""

    def __init__(self, A, space, order, block=2):
        import ctypes as C
        from . import _lib
        A = A.tocsr()
        n = A.shape[0]
        self.n = n
        order = np.asarray(order, dtype=np.int64)
        blk = element_block_ids(space.mesh, block)[space.dof_owner_elem]
        new2old = order[np.argsort(blk[order], kind="stable")]
        bnew = blk[new2old]
        Ap = A[new2old][:, new2old].tocoo()
        keep = bnew[Ap.row] == bnew[Ap.col]
        F = sp.csr_matrix((Ap.data[keep], (Ap.row[keep], Ap.col[keep])), shape=(n, n))
        F.sort_indices()
        data = F.data.astype(np.float64, copy=True)
        fail = vec.ilu0_factor_host(F.indptr, F.indices, data)
        self.jacobi = None
        if fail >= 0:
            diag = A.diagonal().copy()
            diag[diag == 0.0] = 1.0
            self.jacobi = 0.6 / diag
            self._jac = dev.to_device(self.jacobi)
            return
        starts = np.flatnonzero(np.r_[True, bnew[1:] != bnew[:-1]])
        block_ptr = np.r_[starts, n].astype(np.int64)
        self.nblocks = len(starts)
        ip = np.ascontiguousarray(F.indptr, dtype=np.int64)
        ix = np.ascontiguousarray(F.indices, dtype=np.int64)
        n2o = np.ascontiguousarray(new2old, dtype=np.int64)
        h = C.c_void_p()
        _lib.check(_lib.lib.fb_blockilu_create(n, self.nblocks, _lib.ptr(block_ptr), _lib.ptr(n2o),
                                               _lib.ptr(ip), _lib.ptr(ix), _lib.ptr(data),
                                               C.byref(h)))
        self.handle = h
        self._lib = _lib

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and self._lib is not None and self._lib.lib is not None:
            self._lib.lib.fb_blockilu_destroy(h)

    def _apply(self, r, out, transpose, stream):
        if self.jacobi is not None:
            return vec.vmul(self._jac, r, out, stream)
        self._lib.check(self._lib.lib.fb_blockilu_apply(
            self.handle, int(transpose), r.data_ptr(), out.data_ptr(),
            dev.stream_handle() if stream is None else stream))
        return out

    def forward_into(self, r, out, stream=None):
        return self._apply(r, out, False, stream)

    def backward_into(self, r, out, stream=None):
        return self._apply(r, out, True, stream)

    @property
    def adds_in_place(self):
        """True when backward_add_into is available (level-packed sweeps)."""
        if getattr(self, "_adds", None) is None:
            self._adds = (self.jacobi is None and getattr(self, "handle", None) is not None
                          and self._lib.lib.fb_blockilu_sweep_kind(self.handle) == 2)
        return self._adds

    def backward_add_into(self, r, out, stream=None):
        """out += (LU)^-T r in the sweep's final store (bitwise backward_into
        followed by axpby(1, t, 1, out))."""
        self._lib.check(self._lib.lib.fb_blockilu_apply_add(
            self.handle, 1, r.data_ptr(), out.data_ptr(),
            dev.stream_handle() if stream is None else stream))
        return out

    forward = ILU0Smoother.forward
    backward = ILU0Smoother.backward


class DenseInverseSolver:
    """Coarse direct solve through a dense inverse computed once on the
    device (cuSOLVER via torch.linalg.inv); applied with a deterministic
    libfbb200 matrix-vector kernel.  Used for coarse levels up to ~20k rows."""

    def __init__(self, A):
        from . import _lib
        self.n = A.shape[0]
        M = torch.from_numpy(np.asarray(A.toarray(), dtype=np.float64)).to(dev.device())
        self.inv = torch.linalg.inv(M).contiguous()
        del M
        self._lib = _lib

    def solve_into(self, b, x, stream=None):
        self._lib.check(self._lib.lib.fb_dense_mv(self.n, self.inv.data_ptr(), b.data_ptr(),
                                                  x.data_ptr(),
                                                  dev.stream_handle() if stream is None else stream))
        return x

    def solve(self, b):
        bd, host = dev.DeviceIn.get(b)
        out = torch.empty_like(bd)
        self.solve_into(bd, out)
        return dev.to_host(out) if host else out


class SparseLUSolver:
    """Coarse direct solve: host sparse LU (SuperLU via scipy, COLAMD, as the
    reference's splu at solvers.py:372), device triangular solves."""

    def __init__(self, A):
        A = A.tocsc()
        self.n = A.shape[0]
        lu = spla.splu(A)
        self.lu = lu
        self._L = vec.TriSolve(lu.L.tocsr(), lower=True, unit_diag=True)
        self._U = vec.TriSolve(lu.U.tocsr(), lower=False, unit_diag=False)
        self._pr = torch.from_numpy(lu.perm_r.astype(np.int32)).to(dev.device())
        self._pc = torch.from_numpy(lu.perm_c.astype(np.int32)).to(dev.device())
        self._a = dev.empty(self.n)
        self._b = dev.empty(self.n)

    def solve_into(self, b, x, stream=None):
        # Pr A Pc = L U:  x = Pc U^-1 L^-1 Pr b
        vec.permute(self._pr, b, self._a, scatter=True, stream=stream)
        self._L.solve_into(self._a, self._b, stream)
        self._U.solve_into(self._b, self._a, stream)
        return vec.permute(self._pc, self._a, x, scatter=False, stream=stream)

    def solve(self, b):
        bd, host = dev.DeviceIn.get(b)
        out = torch.empty_like(bd)
        self.solve_into(bd, out)
        return dev.to_host(out) if host else out


class LORPreconditioner(_DeviceMixin):
    """Degree-ladder V(1,1) cycle on LOR matrices (solvers.py:321-392), applied
    on the device: per level one ILU(0) forward sweep, residual SpMV, P^T
    restriction, recursive correction, P prolongation, residual SpMV, ILU(0)
    backward sweep; the Q1 bottom level is an exact direct solve.

    smoother="block" (default for stiffness / Helmholtz): block-Jacobi ILU(0)
    over element cubes of `block`^d elements (default 2) in
    first-touch order -- one launch per sweep, +0/+1 iterations vs the
    reference (SURVEY 8(e'), tests/test_gpu_solvers.py).  Mass defaults to
    the global smoother.  smoother="global": the
    reference's global first-touch ILU(0), reproduced to rounding (its
    triangular solves are a dependency chain of ~60 n levels).
    coarse="auto": dense inverse up to 20k coarse rows, else sparse LU."""

    def __init__(self, space, kind, nu=1.0, c=0.0, dirichlet_attrs=None,
                 pure_neumann=False, backend=None, smoother=None, block=None, coarse="auto"):
        if smoother is None:
            # the Q1 mass LOR matrix loses too much coupling when blocked
            # (37 -> 42 CG iterations on the 3D p=3 golden case); stiffness and
            # Helmholtz stay within +1 of the reference for any block size
            smoother = "global" if kind == "mass" else DEFAULT_SMOOTHER
        if block is None:
            # 2^d-element blocks: +0/+1 iterations at p = 4 and 7 on 1M DoFs
            # (tools/blk_sweep.py); single-element blocks cost +1/+2
            block = 2
        if smoother not in ("block", "global"):
            raise ValueError(f"unknown smoother {smoother!r}")
        if space.vdim != 1:
            raise ValueError("LOR cycles act componentwise on scalar spaces")
        if pure_neumann and dirichlet_attrs is not None:
            raise ValueError("pure-Neumann cycle expects no constrained dofs")
        self.pure_neumann = pure_neumann
        mesh = space.mesh
        self.levels = []
        self.transfers = []
        prev = None
        for deg in lor_mod.degree_ladder(space.p):
            lsp = space if deg == space.p else FESpace(mesh, deg)
            if dirichlet_attrs is None:
                bdr = np.zeros(0, dtype=np.int64)
            elif dirichlet_attrs == "all":
                bdr = lsp.boundary_dof_set()
            else:
                bdr = lsp.boundary_dof_set(dirichlet_attrs)
            A = lor_mod.lor_matrix(lsp, kind, nu=nu, c=c, constrained=bdr)
            if pure_neumann:
                A = lor_mod.constrain_matrix(A, np.array([0], dtype=np.int64))
            self.levels.append((lsp, A))
            if prev is not None:
                self.transfers.append(lor_mod.nodal_interpolation(prev, lsp))
            prev = lsp
        self.A = self.levels[0][1]
        self.smoother_kind = smoother
        if smoother == "global":  # the reference's global first-touch ILU(0)
            self.smoothers = [ILU0Smoother(A, lor_mod.first_touch_ordering(lsp), backend=backend)
                              for lsp, A in self.levels[:-1]]
        else:
            self.smoothers = [BlockILU0Smoother(A, lsp, lor_mod.first_touch_ordering(lsp), block)
                              for lsp, A in self.levels[:-1]]
        Ac = self.levels[-1][1]
        if coarse == "dense" or (coarse == "auto" and Ac.shape[0] <= 20000):
            self._bottom = DenseInverseSolver(Ac)
        else:
            self._bottom = SparseLUSolver(Ac)
        self._A = [vec.DeviceCSR(A) for _, A in self.levels]
        self._P = [vec.DeviceCSR(P) for P in self.transfers]
        self._Pt = [vec.DeviceCSR(P.T.tocsr()) for P in self.transfers]
        sizes = [A.shape[0] for _, A in self.levels]
        self._x = [dev.empty(n) for n in sizes]
        self._r = [dev.empty(n) for n in sizes]
        self._t = [dev.empty(n) for n in sizes]
        self._t2 = [dev.empty(n) for n in sizes]
        self._proj = MeanProjector() if pure_neumann else None

    def _cycle(self, level, r, x, st):
        if level == len(self.levels) - 1:
            self._bottom.solve_into(r, x, st)
            return
        A = self._A[level]
        sm = self.smoothers[level]
        t, t2 = self._t[level], self._t2[level]
        sm.forward_into(r, x, st)
        A.residual_into(r, x, t, st)
        rc, xc = self._r[level + 1], self._x[level + 1]
        self._Pt[level].apply_into(t, rc, st)
        self._cycle(level + 1, rc, xc, st)
        P = self._P[level]
        if hasattr(P, "apply_add_into"):  # structured transfer: x += P xc in one pass
            P.apply_add_into(xc, x, st)
        else:
            P.apply_into(xc, t, st)
            vec.axpby(1.0, t, 1.0, x, st)
        A.residual_into(r, x, t, st)
        if getattr(sm, "adds_in_place", False):  # x += M^-T t in the sweep's store
            sm.backward_add_into(t, x, st)
        else:
            sm.backward_into(t, t2, st)
            vec.axpby(1.0, t2, 1.0, x, st)

    @property
    def graph_safe(self):
        """The V-cycle is device launches only on preallocated level vectors
        (block smoother, or the global ILU whose level-scheduled triangular
        solves capture as plain kernels; dense-inverse or device sparse-LU
        coarse solve; no mean projection)."""
        return (self.smoother_kind in ("block", "global")
                and isinstance(self._bottom, (DenseInverseSolver, SparseLUSolver))
                and not self.pure_neumann)

    def clone_workspace(self):
        """A view of this preconditioner (same matrices, smoothers and coarse
        inverse) with its own level vectors, so several can run concurrently
        on different streams; None when a shared handle keeps state between
        launches (the global ILU's graphs, a sparse-LU coarse solve)."""
        import copy
        if self.smoother_kind != "block" or not isinstance(self._bottom, DenseInverseSolver):
            return None
        c = copy.copy(self)
        if self._proj is not None:  # own projector: its reduction scratch is per stream
            c._proj = _StreamMeanProjector()
        c._x = [dev.empty(t.shape[0]) for t in self._x]
        c._r = [dev.empty(t.shape[0]) for t in self._r]
        c._t = [dev.empty(t.shape[0]) for t in self._t]
        c._t2 = [dev.empty(t.shape[0]) for t in self._t2]
        return c

    def apply_into(self, r, out, stream=None):
        st = dev.stream_handle() if stream is None else stream
        rr = r
        if self.pure_neumann:
            rr = self._r[0]
            self._proj.apply_into(r, rr, st)
        self._cycle(0, rr, out, st)
        if self.pure_neumann:
            self._proj.apply_into(out, out, st)
        return out


class BlockDiagonalPreconditioner(_DeviceMixin):
    """One scalar preconditioner per vector component (solvers.py:395-410)."""

    def __init__(self, scalar_precond, vdim, ndofs_scalar):
        self.inner = scalar_precond
        self.vdim = vdim
        self.ns = ndofs_scalar
        self._apply = _device_apply(scalar_precond)
        # components are independent: with per-component workspaces the
        # (latency-bound) V-cycles run concurrently on their own streams.
        # Only for small components: measured on p = 5 box hierarchies
        # (tools/bd_concurrency.py), 0.5M rows per component 2.0x faster,
        # 1.7M 1.14x, 4.1M even, 13.8M / 32.8M 1.3x / 1.4x SLOWER than one
        # after the other (the three hierarchies then compete for L2 / HBM).
        self._par = None
        par_max = int(os.environ.get("FB_BD_CONCURRENT_MAX", "3000000"))
        if vdim > 1 and hasattr(scalar_precond, "clone_workspace") and ndofs_scalar <= par_max:
            clones = [scalar_precond.clone_workspace() for _ in range(vdim - 1)]
            if all(c is not None for c in clones) and torch.cuda.is_available():
                self._par = [scalar_precond] + clones
                self._streams = [torch.cuda.Stream(device=dev.device()) for _ in range(vdim)]
                self._done = [torch.cuda.Event() for _ in range(vdim)]
                self._fork = torch.cuda.Event()
        # large components one after the other: with one V-cycle for all of
        # them the fine-level residuals share a pass over the level matrix
        self._multi = (self._par is None and vdim > 1
                       and hasattr(scalar_precond, "apply_multi_into")
                       and os.environ.get("FB_BD_MULTI", "1") != "0")
        if self._multi:
            scalar_precond.prepare_multi(vdim)

    @property
    def graph_safe(self):
        """Capturable: the concurrent components fork from and join back into
        the current stream with events (the stream-capture pattern)."""
        return bool(getattr(self.inner, "graph_safe", False))

    def apply_into(self, r, out, stream=None):
        ns = self.ns
        if self._par is not None and stream is None:
            cur = torch.cuda.current_stream()
            self._fork.record(cur)
            for c, (pc, s) in enumerate(zip(self._par, self._streams)):
                s.wait_event(self._fork)
                pc.apply_into(r[c * ns:(c + 1) * ns], out[c * ns:(c + 1) * ns], s.cuda_stream)
                self._done[c].record(s)
            for e in self._done:
                cur.wait_event(e)
            return out
        if self._multi:
            return self.inner.apply_multi_into(r, out, self.vdim, ns, stream)
        for c in range(self.vdim):
            self._apply(r[c * ns:(c + 1) * ns], out[c * ns:(c + 1) * ns])
        return out


class InnerCG(_DeviceMixin):
    """Fixed-iteration CG used as a preconditioner (solvers.py:413-425)."""

    def __init__(self, A, precond=None, iterations=3):
        self.A = A
        self.precond = precond
        self.cfg = SolverConfig(rel_tol=0.0, max_iters=iterations)

    def apply_into(self, r, out, stream=None):
        x, _ = cg(self.A, r, precond=self.precond, config=self.cfg)
        out.copy_(x)
        return out
