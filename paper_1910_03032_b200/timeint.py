"""Projection (velocity-correction) stepping on the device: the cfg5 caller.

Mirrors the reference's ``ProjectionStepper`` (timeint.py:218-388) and its
BDF/extrapolation coefficients (timeint.py:102-135): explicit extrapolated
convection, a pressure Poisson solve with the LOR V-cycle (pure Neumann,
mean-projected CG), an implicit vector Helmholtz solve with a per-component
LOR V-cycle, and a mass solve for the nodal convection term.  Every operator
(mass, convection, gradient and its transpose, stiffness, Helmholtz) and every
solver runs through libfbb200; the state and the history vectors live on the
device and the BDF combinations are libfbb200 axpby kernels.

Periodic domains (the Taylor-Green vortex of cfg5) and bounded ones: with
boundary faces the step adds the reference's surface functionals
(``boundary_rotational_rhs`` / ``boundary_normal_flux``, mfop.py:623-807; both
device SpMVs of face matrices built once, ``boundary.py``), Dirichlet
velocity lifting and a constrained Helmholtz solve with a Dirichlet LOR
V-cycle (timeint.py:266-269, 310-316, 338-381).
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import boundary
from . import device as dev
from . import mfop, vec
from .solvers import (BlockDiagonalPreconditioner, DiagonalPreconditioner, LORPreconditioner,
                      MeanProjector, SolverConfig, cg, collocated_mass_diagonal, deflate_mean)
from .spaces import FESpace


@dataclass(frozen=True)
class BDFScheme:
    """BDF differentiation weights b and extrapolation weights a of order k."""

    k: int
    b: np.ndarray
    a: np.ndarray


_BDF_B = {1: (1.0, -1.0), 2: (1.5, -2.0, 0.5), 3: (11.0 / 6.0, -3.0, 1.5, -1.0 / 3.0)}
_EXT_A = {1: (1.0,), 2: (2.0, -1.0), 3: (3.0, -3.0, 1.0)}


def bdf_coefficients(k):
    """BDF-k / EXT-k weights (timeint.py:119-135), checked on polynomials."""
    if k not in _BDF_B:
        raise ValueError(f"BDF order must be 1, 2, or 3, got {k}")
    s = BDFScheme(k, np.array(_BDF_B[k]), np.array(_EXT_A[k]))
    for m in range(k + 1):
        val = sum(s.b[j] * (-float(j)) ** m for j in range(k + 1))
        if abs(val - (1.0 if m == 1 else 0.0)) > 1e-12:
            raise AssertionError(f"BDF{k} fails on t^{m}")
    for m in range(k):
        val = sum(s.a[j - 1] * (-float(j)) ** m for j in range(1, k + 1))
        if abs(val - (0.0 ** m if m else 1.0)) > 1e-12:
            raise AssertionError(f"extrapolation of order {k} fails on t^{m}")
    return s


@dataclass
class StepReport:
    """Iteration counts of the sub-solves in one projection step."""

    t: float
    mass_iters: int = 0
    pressure_iters: int = 0
    helmholtz_iters: int = 0
    phase_ms: dict = None  # device time per phase when the stepper's `profile` is set


def _combo(terms, n):
    """sum_j c_j v_j of device vectors with libfbb200 axpby kernels."""
    out = dev.zeros(n)
    for c, v in terms:
        vec.axpby(float(c), v, 1.0, out)
    return out


class ProjectionStepper:
    """BDF-k / extrapolation velocity-correction stepping for Navier-Stokes
    (timeint.py:218-388) with device-resident state."""

    def __init__(self, vspace, pspace, geom, k, dt, nu, forcing=None, dirichlet=None,
                 config=None, smoother=None):
        if pspace.p != vspace.p or pspace.vdim != 1:
            raise ValueError("projection expects scalar pressure of equal degree")
        if vspace.vdim != vspace.dim:
            raise ValueError("velocity space must have vdim == dim")
        self.k = int(k)
        if self.k not in (1, 2, 3):
            raise ValueError("projection order must be 1, 2, or 3")
        mesh = vspace.mesh
        self.has_boundary = mesh.boundary_faces.shape[0] > 0
        self.dt = float(dt)
        self.nu = float(nu)
        self.vspace, self.pspace, self.geom = vspace, pspace, geom
        self.forcing = forcing
        self.dirichlet = dirichlet
        self.config = config or SolverConfig(rel_tol=1e-10, max_iters=400)
        self.smoother = smoother

        self.M = mfop.MassOperator(vspace, geom)
        self.conv = mfop.ConvectionOperator(vspace, geom)
        self.G = mfop.GradientOperator(vspace, pspace, geom)
        self.D = mfop.DivergenceOperator(vspace, pspace, geom)
        self.Lp = mfop.StiffnessOperator(pspace, geom)
        self.mass_pre = DiagonalPreconditioner(collocated_mass_diagonal(vspace))
        self.pressure_pre = self._pressure_cycle()
        self.mean = MeanProjector()
        self.pressure_weights = collocated_mass_diagonal(pspace)
        self.bdofs = (vspace.expand_dofs(vspace.boundary_dof_set())
                      if self.has_boundary else np.zeros(0, dtype=np.int64))
        self._bdofs_dev = torch.from_numpy(self.bdofs).to(dev.device()) if self.has_boundary else None
        self._helm = {}
        self._scalar_v = self._scalar_velocity_space()
        self.t = None
        self.u = None
        self.p = None
        self.u_hist, self.n_hist, self.r_hist = [], [], []
        self._volume = self._domain_volume()

    # -- preconditioner / space factories (overridden by the scale-mode stepper) --

    def _pressure_cycle(self):
        return LORPreconditioner(self.pspace, "stiffness", pure_neumann=True,
                                 smoother=self.smoother)

    def _helmholtz_cycle(self, c):
        return LORPreconditioner(self._scalar_v, "helmholtz", nu=self.nu, c=c,
                                 dirichlet_attrs=("all" if self.has_boundary else None),
                                 smoother=self.smoother)

    def _scalar_velocity_space(self):
        return FESpace(self.vspace.mesh, self.vspace.p)

    def _domain_volume(self):
        return float(np.sum(self.geom.detj @ self.geom.w))

    # -- state ----------------------------------------------------------------

    def initialize(self, u0, t0=0.0):
        self.t = float(t0)
        self.u = dev.to_device(np.asarray(u0, dtype=np.float64)).clone()
        self.p = dev.zeros(self.pspace.ndofs)
        self.u_hist = [self.u.clone()]
        self.n_hist = [self._nodal_convection(self.u)[0]]
        self.r_hist = [self._rotational_bc(self.u)]
        return self

    def initialize_history(self, states, t_last):
        """Full-order start from k states ordered oldest to newest
        (timeint.py:280-294)."""
        if len(states) != self.k:
            raise ValueError(f"need {self.k} states, got {len(states)}")
        self.t = float(t_last)
        self.u_hist, self.n_hist, self.r_hist = [], [], []
        for u in states:
            u = dev.to_device(np.asarray(u, dtype=np.float64)).clone()
            self.u_hist.insert(0, u)
            self.n_hist.insert(0, self._nodal_convection(u)[0])
            self.r_hist.insert(0, self._rotational_bc(u))
        self.u = self.u_hist[0].clone()
        self.p = dev.zeros(self.pspace.ndofs)
        return self

    # -- pieces ----------------------------------------------------------------

    def _mass_solve(self, rhs):
        tol = min(1e-12, self.config.rel_tol)
        x, rep = cg(self.M, rhs, precond=self.mass_pre,
                    config=SolverConfig(rel_tol=tol, max_iters=300))
        if not rep.converged:
            raise RuntimeError(f"mass solve failed: {rep}")
        return x, rep.iterations

    def _nodal_convection(self, u):
        y = self.conv.apply(u)
        vec.scale(-1.0, y, y)
        return self._mass_solve(y)

    def _rotational_bc(self, u):
        """-nu (n x curl u, grad q) on the boundary (timeint.py:310-316)."""
        if not self.has_boundary:
            return None
        return boundary.boundary_rotational_rhs(self.vspace, self.pspace, u, nu=self.nu)

    def _helmholtz(self, b0):
        key = round(b0, 12)
        if key not in self._helm:
            # one Helmholtz system at a time: the start-up orders (BDF1, BDF2)
            # use theirs once, and each holds a full LOR hierarchy
            self._helm.clear()
            import gc
            gc.collect()
            c = b0 / self.dt
            op = mfop.HelmholtzOperator(self.vspace, self.geom, c=c, nu=self.nu)
            A = mfop.ConstrainedOperator(op, self.bdofs)
            cyc = self._helmholtz_cycle(c)
            pre = BlockDiagonalPreconditioner(cyc, self.vspace.vdim, self.vspace.ndofs_scalar)
            self._helm[key] = (op, A, pre)
        return self._helm[key]

    def _forcing_nodal(self, t):
        if self.forcing is None:
            return None
        return dev.to_device(self.vspace.project(lambda x: self.forcing(x, t)))

    # -- one step ----------------------------------------------------------------

    def step(self):
        """Advance to t + dt (timeint.py:338-381); returns a StepReport."""
        if self.t is None:
            raise RuntimeError("stepper not initialized")
        k_eff = min(self.k, len(self.u_hist))
        s = bdf_coefficients(k_eff)
        dt, t_new = self.dt, self.t + self.dt
        b0 = s.b[0]
        rep = StepReport(t=t_new)
        marks = []

        def mark(name):  # CUDA events between phases (profile mode only)
            if getattr(self, "profile", False):
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                marks.append((name, e))

        mark("start")
        nv = self.vspace.ndofs
        terms = [(-s.b[j] / dt, self.u_hist[j - 1]) for j in range(1, k_eff + 1)]
        terms += [(s.a[j - 1], self.n_hist[j - 1]) for j in range(1, k_eff + 1)]
        f_star = self._forcing_nodal(t_new)
        if f_star is not None:
            terms.insert(0, (1.0, f_star))
        F = _combo(terms, nv)

        g_new = (None if self.dirichlet is None or not self.has_boundary
                 else (lambda x: self.dirichlet(x, t_new)))
        rhs_p = self.G.apply_transpose(F)
        if self.has_boundary:
            for j in range(1, k_eff + 1):
                vec.axpby(float(s.a[j - 1]), self.r_hist[j - 1], 1.0, rhs_p)
            if g_new is not None:
                fl = boundary.flux_matrix(self.pspace)(g_new)  # device SpMV
                vec.axpby(-(b0 / dt), fl, 1.0, rhs_p)
        rhs_p = deflate_mean(rhs_p)
        mark("rhs")
        p, prep = cg(self.Lp, rhs_p, precond=self.pressure_pre, x0=self.p, project=self.mean,
                     config=self.config)
        mark("pressure_solve")
        if not prep.converged:
            raise RuntimeError(f"pressure solve failed: {prep}")
        rep.pressure_iters = prep.iterations

        op, A, pre = self._helmholtz(b0)
        b_u = self.M.apply(F)
        vec.axpby(-1.0, self.G.apply(p), 1.0, b_u)
        u_lift = None
        if g_new is not None:
            lift = np.zeros(nv)
            lift[self.bdofs] = self.vspace.project(g_new)[self.bdofs]
            u_lift = dev.to_device(lift)
            vec.axpby(-1.0, op.apply(u_lift), 1.0, b_u)
        if self.has_boundary:
            b_u.index_fill_(0, self._bdofs_dev, 0.0)
        mark("velocity_rhs")
        u, hrep = cg(A, b_u, precond=pre, config=self.config)
        mark("helmholtz_solve")
        if not hrep.converged:
            raise RuntimeError(f"velocity solve failed: {hrep}")
        rep.helmholtz_iters = hrep.iterations
        if u_lift is not None:
            vec.axpby(1.0, u_lift, 1.0, u)

        n_new, it_n = self._nodal_convection(u)
        rep.mass_iters = it_n
        mark("convection_mass_solve")
        if marks:
            torch.cuda.synchronize()
            rep.phase_ms = {n1: round(e0.elapsed_time(e1), 3)
                            for (_, e0), (n1, e1) in zip(marks[:-1], marks[1:])}
        self.u_hist.insert(0, u)
        self.n_hist.insert(0, n_new)
        self.r_hist.insert(0, self._rotational_bc(u))
        del self.u_hist[self.k:], self.n_hist[self.k:], self.r_hist[self.k:]
        self.u, self.p, self.t = u, deflate_mean(p, self.pressure_weights), t_new
        return rep

    def kinetic_energy(self, u=None):
        """Volume-averaged kinetic energy u' M u / (2 |Omega|)."""
        v = self.u if u is None else u
        return float(vec.dot(v, self.M.apply(v))) / (2.0 * self._volume)

    def divergence_residual(self, u=None):
        """Euclidean norm of the weak divergence of the current velocity
        (timeint.py:397-400).  u may be a host array or a device tensor."""
        v = self.u if u is None else dev.to_device(u)
        w = self.D.apply(v)
        return float(torch.linalg.norm(w)) if torch.is_tensor(w) else float(np.linalg.norm(w))

    def state_host(self):
        """(u, p) as host numpy arrays -- the reference stepper's `u` / `p`
        attributes are numpy; here they stay device tensors between steps."""
        return dev.to_host(self.u), dev.to_host(self.p)


class BoxProjectionStepper(ProjectionStepper):
    """The projection stepper in scale mode (cfg5 at size on one GPU): a
    periodic (or bounded, Dirichlet) structured box with the block-major
    `structured.BoxSpace` numbering, factors built on the device and the
    pressure / Helmholtz LOR hierarchies assembled and factored on the device
    (`structured.BoxLORPreconditioner`: block-ILU smoother, pure-Neumann pin
    + mean projection for the pressure).  Same step as ProjectionStepper
    (timeint.py:338-388); the velocity is SoA over the box numbering."""

    def __init__(self, mesh, p, k, dt, nu, forcing=None, config=None, block=2):
        from . import geometry, structured
        ddev = dev.device()
        if any(not a for a in mesh.periodic):
            raise ValueError("BoxProjectionStepper supports fully periodic boxes")
        self._block = block
        vspace = structured.BoxSpace(mesh, p, block=block, device=ddev, vdim=3)
        pspace = structured.BoxSpace(mesh, p, block=block, device=ddev)
        geom = geometry.DeviceGeometry(mesh, vspace.basis.quad)
        super().__init__(vspace, pspace, geom, k, dt, nu, forcing=forcing, config=config)

    def _pressure_cycle(self):
        from . import structured
        return structured.BoxLORPreconditioner(self.pspace, "stiffness", dirichlet_attrs=None,
                                               pure_neumann=True, block=self._block)

    def _helmholtz_cycle(self, c):
        from . import structured
        return structured.BoxLORPreconditioner(self._scalar_v, "helmholtz", nu=self.nu, c=c,
                                               block=self._block)

    def _scalar_velocity_space(self):
        return self.pspace  # same degree, same box numbering

    def _domain_volume(self):
        from .geometry import compute_geometric_factors
        from .quadrature import GAUSS_LEGENDRE, quadrature_rule
        g = compute_geometric_factors(self.vspace.mesh, quadrature_rule(GAUSS_LEGENDRE, 2))
        return float(np.sum(g.detj @ g.w))
