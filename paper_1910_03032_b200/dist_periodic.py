"""Multi-GPU scale mode on PERIODIC boxes (the cfg5 Taylor-Green domain):
z-slabs on a ring.

`dist_box` shards Dirichlet boxes: a slab's lower cut plane belongs to the rank
below, and the last rank owns the top of the box.  On a periodic box
(mesh.py:81-96) the lattice has n_z p planes and plane n_z p is plane 0, so
the slabs form a ring: rank r owns the planes (e0 p, e1 p] (rank 0 also
plane 0; the last rank's top element plane is rank 0's plane 0).  Every rank
keeps two ghost planes, uniform around the ring:

* lower ghost: the plane below its lowest owned plane (rank 0: plane
  n_z p - 1, owned by the last rank; others: plane e0 p, owned by rank-1);
* upper ghost: the plane above its highest owned plane (the last rank:
  plane 0, owned by rank 0; others: plane e1 p + 1, owned by rank+1).

A ghost update sends every rank's top owned plane up and its bottom-most
neighbour-facing plane down (`exchange_ring`, periodic neighbours); the
operator's cut-plane partial sums go down from every rank but 0, and up from
the last rank into rank 0's plane 0.  x and y wrap inside each slab.  The
level objects mirror `dist_box.SlabLevel`, so the sharded operator
(`dist_box.DistOperator`), the block-Jacobi ILU(0) (same blocks as one GPU:
identical factor) and the V-cycle recursion are shared; the Q1 problem is
agglomerated and solved by the periodic `structured.BoxLORPreconditioner`
(pure-Neumann pin + mean projection for the pressure).
"""

import ctypes as C

import numpy as np
import torch

from . import _lib
from . import device as dev
from . import geometry
from . import lor as lor_mod
from . import mfop
from . import solvers
from . import structured as S
from . import vec
from .dist_box import DistOperator, slab_layers
from .quadrature import build_eval_matrices, make_basis

PER = (True, True, True)


def _plane_ids(counts, p, block, g, device):
    """Global ids of lattice plane g of the periodic box, (Ny, Nx)."""
    ids, _ = S.box_lattice_ids(counts, p, block, device, gz_range=(g, g + 1), periodic=PER)
    return ids[0]


def _layers_mesh(mesh, layers):
    """A mesh holding the given global element layers (in order, wrapping)."""
    nx, ny, nz = mesh.counts
    plane = nx * ny
    corners = np.concatenate([mesh.corners[L * plane:(L + 1) * plane] for L in layers])
    cm = geometry.cartesian_mesh((nx, ny, len(layers)))
    return geometry.Mesh(3, cm.vertices, cm.elements, corners, cm.boundary_faces,
                         (True, True, False), (nx, ny, len(layers)))


class PeriodicSlabLevel:
    """Rank r's view of one level (degree p, smoother blocks of `block`
    elements) of a periodic box split into z-slabs on a ring.  Local vectors
    are [owned | lower ghost plane | upper ghost plane]."""

    def __init__(self, mesh, p, block, layers, rank, world, device):
        if tuple(mesh.periodic) != PER:
            raise ValueError("PeriodicSlabLevel needs a fully periodic box")
        if world < 2:
            raise ValueError("a ring needs at least two ranks (one GPU: structured.BoxSpace)")
        self.gmesh, self.p, self.block = mesh, p, block
        self.rank, self.world = rank, world
        nx, ny, nz = (int(c) for c in mesh.counts)
        self.counts = (nx, ny, nz)
        e0, e1 = layers[rank]
        if e0 % block or e1 % block:
            raise ValueError("slab bounds must align with smoother blocks")
        self.e0, self.e1 = e0, e1
        self.first, self.last = rank == 0, rank == world - 1
        Nx, Ny, Nz = nx * p, ny * p, nz * p
        self.P = Nx * Ny
        nbx, nby = -(-nx // block), -(-ny // block)
        _, bptr = S.box_lattice_ids((nx, ny, nz), p, block, torch.device("cpu"),
                                    gz_range=(0, 1), periodic=PER)
        b0, b1 = (e0 // block) * nby * nbx, (e1 // block) * nby * nbx
        self.off, self.n_own = int(bptr[b0]), int(bptr[b1] - bptr[b0])
        self.block_ptr = bptr[b0:b1 + 1] - bptr[b0]
        self.lower, self.upper = self.n_own, self.n_own + self.P
        self.n_local = self.n_own + 2 * self.P
        self.low_plane = (Nz - 1) if self.first else e0 * p
        self.up_plane = 0 if self.last else e1 * p + 1
        pidx = torch.arange(self.P, device=device, dtype=torch.int64).view(Ny, Nx)
        self.ghost_gids = {}

        def local_plane(g):
            gg = g % Nz
            ids = _plane_ids((nx, ny, nz), p, block, gg, device)
            loc = ids - self.off
            own = (loc >= 0) & (loc < self.n_own)
            out = torch.full_like(loc, -1)
            out = torch.where(own, loc, out)
            if gg == self.low_plane:
                out = torch.where(own, out, self.lower + pidx)
                self.ghost_gids["lower"] = ids.reshape(-1)
            elif gg == self.up_plane:
                out = torch.where(own, out, self.upper + pidx)
                self.ghost_gids["upper"] = ids.reshape(-1)
            return out

        # element lattice of the slab (planes e0 p .. e1 p; the last rank's top wraps)
        elem = torch.stack([local_plane(g) for g in range(e0 * p, e1 * p + 1)])
        if int((elem < 0).sum()) != 0:
            raise RuntimeError("unmapped lattice point in the slab")
        self.lid_elems = elem.to(torch.int32).contiguous()
        # LOR rows of the owned planes: the slab's layers plus the layer below
        # (rank 0: the last layer, wrapped) or above (all but the last rank)
        ext = list(range(e0, e1)) + ([] if self.last else [e1])
        if self.first:
            ext = [nz - 1] + ext
        self.ext_layers = ext
        g0 = ext[0] * p if not self.first else (e0 - 1) * p
        planes = [local_plane(g) for g in range(g0, g0 + len(ext) * p + 1)]
        self.lid_ext = torch.stack(planes).to(torch.int32).contiguous()
        self.mesh_ext = _layers_mesh(mesh, [L % nz for L in ext])
        self.mesh_elems = _layers_mesh(mesh, list(range(e0, e1)))
        self.mesh = self.mesh_elems
        # ring send lists: the top owned plane goes up, the neighbour-facing
        # bottom plane (rank 0: plane 0, else plane e0 p + 1) goes down
        top = (Nz - 1) if self.last else e1 * p
        bot = 0 if self.first else e0 * p + 1
        self.send_up_ids = local_plane(top).reshape(-1).to(torch.int32).contiguous()
        self.send_down_ids = local_plane(bot).reshape(-1).to(torch.int32).contiguous()
        self.dim, self.vdim = 3, 1
        self.basis = make_basis(p)
        self.device = device
        self._buf = {}

    # -- space-like interface for the operator / restriction ---------------------
    @property
    def ndofs_scalar(self):
        return self.n_local

    @property
    def ndofs(self):
        return self.n_local

    @property
    def element_dofs(self):
        if "ed" not in self._buf:
            ed = S.lattice_element_dofs(self.lid_elems, self.p, (True, True, False))
            self._buf["ed"] = ed.to(torch.int64).cpu().numpy()
        return self._buf["ed"]

    def boundary_local(self):
        return np.zeros(0, dtype=np.int64)

    def buf(self, name, n):
        t = self._buf.get(name)
        if t is None or t.shape[0] != n:
            t = self._buf[name] = torch.empty(n, dtype=torch.float64, device=self.device)
        return t

    # -- halo operations -----------------------------------------------------------
    def ghost_update(self, comm, x, top1=True):
        """Both ghost planes from their owners around the ring."""
        P = self.P
        su, sd = self.buf("su", P), self.buf("sd", P)
        vec.permute(self.send_up_ids, x, su)
        vec.permute(self.send_down_ids, x, sd)
        comm.exchange_ring(sd, su, x[self.lower:self.lower + P], x[self.upper:self.upper + P])

    def sum_planes(self, comm, y):
        """Cut-plane partial sums: the lower ghost's partials go down (all but
        rank 0), the last rank's upper ghost partials go up into rank 0's
        plane 0; received partials are added to the owned planes."""
        P = self.P
        send_down = y[self.lower:self.lower + P] if not self.first else None
        send_up = y[self.upper:self.upper + P] if self.last else None
        recv_up = self.buf("ru", P) if not self.last else None
        recv_down = self.buf("rd", P) if self.first else None
        comm.exchange_ring(send_down, send_up, recv_down, recv_up)
        st = dev.stream_handle()
        if recv_up is not None:
            _lib.check(_lib.lib.fb_index_add(P, self.send_up_ids.data_ptr(), recv_up.data_ptr(),
                                             y.data_ptr(), st))
        if recv_down is not None:
            _lib.check(_lib.lib.fb_index_add(P, self.send_down_ids.data_ptr(),
                                             recv_down.data_ptr(), y.data_ptr(), st))

    def zero_ghosts(self, y):
        y[self.n_own:].zero_()


class PeriodicLevelMatrix(vec.DeviceCSR):
    """Owned rows of a level's LOR matrix (complete), columns owned + ghosts;
    pure-Neumann levels pin the global DoF 0 (solvers.py:361-362)."""

    def __init__(self, level, kind, nu, c, pin=False):
        lv = level
        corners = torch.from_numpy(np.ascontiguousarray(lv.mesh_ext.corners, dtype=np.float64))
        corners = corners.to(dev.device())
        counts = np.asarray(lv.mesh_ext.counts, dtype=np.int64)
        nodes = np.ascontiguousarray(lv.basis.nodes, dtype=np.float64)
        mask = 64 | 128  # x, y periodic inside the slab; z handled by the extended lattice
        h = C.c_void_p()
        _lib.check(_lib.lib.fb_lor_assemble_box_rows(
            lv.p, _lib.ptr(counts), corners.data_ptr(), _lib.ptr(nodes), lv.lid_ext.data_ptr(),
            _lib.KIND[kind], float(nu), float(c), mask, lv.n_own, lv.n_local, C.byref(h)))
        self.handle = h
        self.shape = (lv.n_own, lv.n_local)
        if pin:  # global DoF 0 = lattice (0, 0, 0): rank 0's local 0, the last rank's upper ghost
            loc = 0 if lv.first else (lv.upper if lv.last else None)
            if loc is not None:
                _lib.check(_lib.lib.fb_csr_pin(h, int(loc)))


class PeriodicTransfer(S.BoxTransfer):
    """p-transfer between two ring slab levels of the same mesh slab."""

    def __init__(self, fine, coarse):
        self.fine_r = mfop.restriction(fine)
        self.hmap_r = mfop.restriction(coarse)
        B1, _ = build_eval_matrices(coarse.basis.nodes, fine.basis.nodes)
        W = np.ascontiguousarray(B1, dtype=np.float64)[None]
        nx, ny, nz = fine.counts
        counts = np.asarray([nx, ny, fine.e1 - fine.e0], dtype=np.int64)
        widx = np.zeros(int(counts.sum()), dtype=np.int64)
        h = C.c_void_p()
        _lib.check(_lib.lib.fb_transfer_create(self.fine_r.handle, self.hmap_r.handle,
                                               _lib.ptr(counts), 1, _lib.ptr(W), _lib.ptr(widx),
                                               C.byref(h)))
        self.handle = h
        _lib.check(_lib.lib.fb_transfer_set_origin(h, 0, 0, fine.e0))
        _lib.check(_lib.lib.fb_transfer_set_periodic(h, 7, nx, ny, nz))


class DistMean:
    """MeanProjector over the ring's owned slices: v - mean(v)."""

    def __init__(self, comm, n_own, n_global):
        self.comm, self.n_own, self.n_global = comm, n_own, float(n_global)
        self._s = dev.zeros(1)
        self._ones = None

    def apply_into(self, v, out, stream=None):
        if self._ones is None:
            self._ones = torch.ones(self.n_own, dtype=torch.float64, device=v.device)
        vec.dot_into(self._ones, v[:self.n_own], self._s)
        self.comm.allreduce_sum(self._s)
        vec.shift_ratio(v, self._s, self.n_global, out)
        return out


class DistPeriodicLOR:
    """Sharded scale-mode V(1,1) cycle on a periodic ring of slabs (same
    recursion as solvers.LORPreconditioner._cycle, solvers.py:375-392); the
    Q1 problem agglomerated and solved by the periodic BoxLORPreconditioner;
    pure_neumann: pinned levels + mean projection before and after."""

    def __init__(self, mesh, p, kind, comm, layers, nu=1.0, c=0.0, block=2, q1_block=4,
                 pure_neumann=False, levels=None):
        self.comm = comm
        r, w = comm.rank, comm.world
        ddev = dev.device()
        degs = [d for d in lor_mod.degree_ladder(p) if d > 1]
        self.levels = levels or [PeriodicSlabLevel(mesh, d, block, layers, r, w, ddev)
                                 for d in degs]
        self.q1 = PeriodicSlabLevel(mesh, 1, q1_block, layers, r, w, ddev)
        self.pure_neumann = pure_neumann
        self._A = [PeriodicLevelMatrix(lv, kind, nu, c, pin=pure_neumann) for lv in self.levels]
        self.smoothers = [S.DeviceBlockILU0(A, lv.block_ptr) for A, lv in zip(self._A, self.levels)]
        chain = self.levels + [self.q1]
        self.transfers = [PeriodicTransfer(chain[i], chain[i + 1]) for i in range(len(self.levels))]
        q1space = S.BoxSpace(mesh, 1, block=q1_block, device=ddev)
        self.coarse = S.BoxLORPreconditioner(q1space, kind, nu=nu, c=c, q1_block=q1_block,
                                             dirichlet_attrs=None if pure_neumann else "all",
                                             pure_neumann=pure_neumann)
        sizes = torch.tensor([self.q1.n_own], dtype=torch.float64, device=ddev)
        allsz = comm.allgather(sizes, [1] * w)
        self.q1_sizes = [int(v) for v in allsz.tolist()]
        self.q1_offsets = np.concatenate([[0], np.cumsum(self.q1_sizes)]).astype(np.int64)
        self._x = [dev.zeros(lv.n_local) for lv in chain]
        self._r = [dev.zeros(lv.n_local) for lv in chain]
        self._t = [dev.zeros(lv.n_local) for lv in chain]
        self._t2 = [dev.zeros(lv.n_local) for lv in chain]
        lv0 = self.levels[0]
        ng = int(np.prod([a * lv0.p for a in lv0.counts]))
        self._proj = DistMean(comm, lv0.n_own, ng) if pure_neumann else None
        self._q1_ghost = None

    def _coarse_solve(self, rq, xq):
        q1 = self.q1
        rg = self.comm.allgather(rq[:q1.n_own], self.q1_sizes)
        xg = torch.empty_like(rg)
        # the Q1 level of the single-GPU cycle (its cycle, not its apply: the
        # mean projection happens once, around the whole V-cycle)
        self.coarse._cycle(0, rg, xg, dev.stream_handle())
        o = int(self.q1_offsets[self.comm.rank])
        vec.copy(xg[o:o + q1.n_own], xq[:q1.n_own])
        if self._q1_ghost is None:
            self._q1_ghost = {k: v.to(torch.int32).contiguous() for k, v in q1.ghost_gids.items()}
        P = q1.P
        vec.permute(self._q1_ghost["lower"], xg, xq[q1.lower:q1.lower + P])
        vec.permute(self._q1_ghost["upper"], xg, xq[q1.upper:q1.upper + P])

    def _cycle(self, i, r, x):
        lv, A, sm = self.levels[i], self._A[i], self.smoothers[i]
        n = lv.n_own
        t, t2 = self._t[i], self._t2[i]
        sm.forward_into(r, x)
        lv.ghost_update(self.comm, x)
        A.residual_into(r, x, t)
        rc, xc = self._r[i + 1], self._x[i + 1]
        T = self.transfers[i]
        cl = self.levels[i + 1] if i + 1 < len(self.levels) else self.q1
        T.restrict_into(t, rc)
        cl.sum_planes(self.comm, rc)
        if i + 1 < len(self.levels):
            self._cycle(i + 1, rc, xc)
            cl.ghost_update(self.comm, xc)
        else:
            self._coarse_solve(rc, xc)
        T.prolong_add_into(xc, x)  # owned x += P xc; ghosts refreshed below
        lv.ghost_update(self.comm, x)
        A.residual_into(r, x, t)
        sm.backward_into(t, t2)
        vec.axpby(1.0, t2[:n], 1.0, x[:n])

    def apply_into(self, r, out, stream=None):
        rr = r
        if self._proj is not None:
            rr = self._r[0]
            self._proj.apply_into(r, rr)
        self._cycle(0, rr, out)
        if self._proj is not None:
            self._proj.apply_into(out, out)
        return out


def dist_cg(A, b, M, comm, n_own, config=None, project=None):
    """solvers.cg with owned-slice dots + all-reduce (and an optional
    distributed projection, e.g. DistMean)."""

    def inner(x, y, out):
        vec.dot_into(x[:n_own], y[:n_own], out)
        comm.allreduce_sum(out)
        return out

    return solvers.cg(A, b, precond=M, config=config, inner=inner, project=project)


def periodic_slab_problem(comm, counts, p, kind="stiffness", c=0.0, nu=1.0, block=2, q1_block=4,
                          pure_neumann=True, rhs_seed=5, mesh=None):
    """One rank's share of a periodic [-pi, pi]^3 solve (cfg5 pressure
    Poisson with pure_neumann, or a Helmholtz solve): sharded operator, ring
    V-cycle, owned slice of the global right-hand side (generated identically
    on every rank; mean-free for the pure-Neumann problem)."""
    r, w = comm.rank, comm.world
    ddev = dev.device()
    mesh = mesh if mesh is not None else geometry.cartesian_mesh(
        counts, lows=(-np.pi,) * 3, highs=(np.pi,) * 3, periodic=PER)
    unit = int(np.lcm(block, q1_block))
    layers = slab_layers(counts[2], w, unit)
    degs = [d for d in lor_mod.degree_ladder(p) if d > 1]
    levels = [PeriodicSlabLevel(mesh, d, block, layers, r, w, ddev) for d in degs]
    lv = levels[0]
    geom = geometry.DeviceGeometry(lv.mesh_elems, lv.basis.quad)
    op_local = mfop.setup(kind, space=lv, geom=geom, nu=nu, c=c)
    A = DistOperator(op_local, lv, comm)
    M = DistPeriodicLOR(mesh, p, kind, comm, layers, nu=nu, c=c, block=block, q1_block=q1_block,
                        pure_neumann=pure_neumann, levels=levels)
    N = int(np.prod([counts[a] * p for a in range(3)]))
    g = torch.Generator(device=ddev)
    g.manual_seed(rhs_seed)
    bg = torch.randn(N, generator=g, dtype=torch.float64, device=ddev)
    if pure_neumann:
        bg -= bg.mean()
    b = dev.zeros(lv.n_local)
    vec.copy(bg[lv.off:lv.off + lv.n_own], b[:lv.n_own])
    proj = DistMean(comm, lv.n_own, N) if pure_neumann else None
    return {"level": lv, "A": A, "M": M, "b": b, "b_global": bg, "project": proj,
            "layers": layers, "mesh": mesh}


# ---------------------------------------------------------------------------
# the projection step on the ring (cfg5 on N GPUs)
# ---------------------------------------------------------------------------

class VectorView:
    """vdim-component view of a ring slab level (SoA, component stride
    n_local): the space-like object the vector operators see."""

    def __init__(self, lv, vdim=3):
        self.lv, self.vdim = lv, vdim
        self.mesh, self.p, self.dim, self.basis = lv.mesh, lv.p, 3, lv.basis
        self.ndofs_scalar = lv.n_local

    @property
    def ndofs(self):
        return self.vdim * self.ndofs_scalar

    @property
    def element_dofs(self):
        return self.lv.element_dofs


class DistFieldOperator:
    """Slab operator between (vector) fields on the ring: ghost update of
    every input component, the local fused kernel, cut-plane partial sums of
    every output component."""

    def __init__(self, apply_local, lv, comm, vin, vout):
        self.apply_local, self.lv, self.comm, self.vin, self.vout = apply_local, lv, comm, vin, vout
        n = lv.n_local
        self.shape = (vout * n, vin * n)

    def apply_into(self, x, y, stream=None):
        lv, n = self.lv, self.lv.n_local
        for c in range(self.vin):
            lv.ghost_update(self.comm, x[c * n:(c + 1) * n])
        self.apply_local(x, y)
        for c in range(self.vout):
            lv.sum_planes(self.comm, y[c * n:(c + 1) * n])
        return y

    def apply(self, x):
        y = dev.empty(self.shape[0])
        return self.apply_into(x, y)


class DistProjectionStepper:
    """ProjectionStepper (timeint.py:218-388) for the periodic Taylor-Green
    box sharded over z-slabs on a ring, one rank per GPU: slab operators
    (mass, convection, G, G^T, D, pressure stiffness, vector Helmholtz) with
    ring halos, distributed CG (owned-slice dots + all-reduce), ring LOR
    V-cycles (pure-Neumann pressure with the distributed mean projection;
    one Helmholtz cycle per velocity component) and the collocated mass
    diagonal assembled with cut-plane sums.  Same step, same preconditioners
    as timeint.BoxProjectionStepper on one GPU."""

    def __init__(self, comm, mesh, p, k, dt, nu, block=2, q1_block=4, config=None):
        from .solvers import DiagonalPreconditioner, SolverConfig, collocated_mass_diagonal
        from .timeint import bdf_coefficients  # noqa: F401 (validated in step)
        self.comm, self.mesh, self.k, self.dt, self.nu = comm, mesh, int(k), float(dt), float(nu)
        self.block, self.q1_block = block, q1_block
        self.config = config or SolverConfig(rel_tol=1e-10, max_iters=400)
        r, w = comm.rank, comm.world
        ddev = dev.device()
        nz = mesh.counts[2]
        self.layers = slab_layers(nz, w, int(np.lcm(block, q1_block)))
        degs = [d for d in lor_mod.degree_ladder(p) if d > 1]
        self.levels = [PeriodicSlabLevel(mesh, d, block, self.layers, r, w, ddev) for d in degs]
        lv = self.lv = self.levels[0]
        self.vv = VectorView(lv, 3)
        n = self.n = lv.n_local
        geom = geometry.DeviceGeometry(lv.mesh_elems, lv.basis.quad)
        self.geom = geom
        M = mfop.MassOperator(self.vv, geom)
        conv = mfop.ConvectionOperator(self.vv, geom)
        G = mfop.GradientOperator(self.vv, lv, geom)
        D = mfop.DivergenceOperator(self.vv, lv, geom)
        Lp = mfop.StiffnessOperator(lv, geom)
        self.M = DistFieldOperator(M.apply_into, lv, comm, 3, 3)
        self.conv = DistFieldOperator(conv.apply_into, lv, comm, 3, 3)
        self.G = DistFieldOperator(G.apply_into, lv, comm, 1, 3)
        self.Gt = DistFieldOperator(G.apply_transpose_into, lv, comm, 3, 1)
        self.D = DistFieldOperator(D.apply_into, lv, comm, 3, 1)
        self.Lp = DistFieldOperator(Lp.apply_into, lv, comm, 1, 1)
        self._ops = (M, conv, G, D, Lp)
        # collocated (GLL) mass diagonal: element sums + cut-plane sums
        dl = dev.to_device(collocated_mass_diagonal(lv))
        lv.sum_planes(comm, dl)
        lv.ghost_update(comm, dl)
        self.pressure_weights = dl
        dh = dl.cpu().numpy()
        self.mass_pre = DiagonalPreconditioner(np.concatenate([dh, dh, dh]))
        N = int(np.prod([a * p for a in mesh.counts]))
        self.N = N
        self.mean = DistMean(comm, lv.n_own, N)
        self.pressure_pre = DistPeriodicLOR(mesh, p, "stiffness", comm, self.layers,
                                            block=block, q1_block=q1_block, pure_neumann=True,
                                            levels=self.levels)
        self._helm = {}
        self._wsum = None
        from .geometry import compute_geometric_factors
        from .quadrature import GAUSS_LEGENDRE, quadrature_rule
        gq = compute_geometric_factors(mesh, quadrature_rule(GAUSS_LEGENDRE, 2))
        self._volume = float(np.sum(gq.detj @ gq.w))
        self.t = self.u = self.p = None
        self.u_hist, self.n_hist = [], []

    # -- distributed reductions ------------------------------------------------------
    def _dot(self, x, y, out, ncomp):
        n, no = self.n, self.lv.n_own
        vec.dot_into(x[:no], y[:no], out)
        if ncomp > 1:
            tmp = dev.zeros(1)
            for c in range(1, ncomp):
                vec.dot_into(x[c * n:c * n + no], y[c * n:c * n + no], tmp)
                vec.axpby(1.0, tmp, 1.0, out)
        self.comm.allreduce_sum(out)
        return out

    def _cg(self, A, b, pre, ncomp, x0=None, project=None):
        return solvers.cg(A, b, precond=pre, config=self.config, x0=x0, project=project,
                          inner=lambda x, y, out: self._dot(x, y, out, ncomp))

    def _weighted_mean_free(self, v):
        """v - (sum w v / sum w): deflate_mean with the collocated weights."""
        no = self.lv.n_own
        w = self.pressure_weights
        if self._wsum is None:
            s = dev.zeros(1)
            vec.dot_into(w[:no], torch.ones(no, dtype=torch.float64, device=w.device), s)
            self.comm.allreduce_sum(s)
            self._wsum = float(s.item())
        num = dev.zeros(1)
        vec.dot_into(w[:no], v[:no], num)
        self.comm.allreduce_sum(num)
        out = torch.empty_like(v)
        vec.shift_ratio(v, num, self._wsum, out)
        return out

    # -- state --------------------------------------------------------------------------
    def scatter_global_velocity(self, u_global):
        """This rank's local velocity (owned slices of the global block-major
        SoA vector, ghosts filled by the first operator apply)."""
        lv, n, ng = self.lv, self.n, self.N
        u = dev.zeros(3 * n)
        ug = dev.to_device(np.asarray(u_global, dtype=np.float64))
        for c in range(3):
            vec.copy(ug[c * ng + lv.off:c * ng + lv.off + lv.n_own], u[c * n:c * n + lv.n_own])
        return u

    def gather_owned(self, v, ncomp):
        n, no = self.n, self.lv.n_own
        parts = [v[c * n:c * n + no] for c in range(ncomp)]
        return [self.comm.allgather(pt, self._sizes()) for pt in parts]

    def _sizes(self):
        if not hasattr(self, "_sz"):
            t = torch.tensor([float(self.lv.n_own)], dtype=torch.float64, device=dev.device())
            self._sz = [int(v) for v in self.comm.allgather(t, [1] * self.comm.world).tolist()]
        return self._sz

    def local_node_coords(self):
        """Physical position of each owned local DoF (first-touch element node,
        as BoxSpace.node_coords); no global vector is formed."""
        from .spaces import element_node_coords
        lv = self.lv
        xyz = element_node_coords(self.vv).reshape(-1, 3)
        ids = np.asarray(lv.element_dofs).reshape(-1)
        out = np.zeros((lv.n_local, 3))
        out[ids[::-1]] = xyz[::-1]  # earliest touching element written last
        return out[:lv.n_own]

    def initialize_from(self, f, t0=0.0):
        """Start from the nodal interpolant of f(x) -> (n, 3), evaluated on
        this rank's owned DoFs only (the bench's 8-GPU path)."""
        vals = np.asarray(f(self.local_node_coords()), dtype=np.float64)
        n, no = self.n, self.lv.n_own
        u = np.zeros(3 * n)
        for c in range(3):
            u[c * n:c * n + no] = vals[:, c]
        return self._start(dev.to_device(u), t0)

    def initialize(self, u_global, t0=0.0):
        return self._start(self.scatter_global_velocity(u_global), t0)

    def _start(self, u, t0):
        self.t = float(t0)
        self.u = u
        self.p = dev.zeros(self.n)
        self.u_hist = [self.u.clone()]
        self.n_hist = [self._nodal_convection(self.u)[0]]
        return self

    def _mass_solve(self, rhs):
        from .solvers import SolverConfig
        tol = min(1e-12, self.config.rel_tol)
        x, rep = solvers.cg(self.M, rhs, precond=self.mass_pre,
                            config=SolverConfig(rel_tol=tol, max_iters=300),
                            inner=lambda a, b, out: self._dot(a, b, out, 3))
        if not rep.converged:
            raise RuntimeError(f"mass solve failed: {rep}")
        return x, rep.iterations

    def _nodal_convection(self, u):
        y = self.conv.apply(u)
        vec.scale(-1.0, y, y)
        return self._mass_solve(y)

    def _helmholtz(self, b0):
        key = round(b0, 12)
        if key not in self._helm:
            # one Helmholtz system at a time: the start-up orders (BDF1, BDF2)
            # use theirs once, and each holds a full LOR hierarchy
            self._helm.clear()
            import gc
            gc.collect()
            c = b0 / self.dt
            op = mfop.HelmholtzOperator(self.vv, self.geom, c=c, nu=self.nu)
            A = DistFieldOperator(op.apply_into, self.lv, self.comm, 3, 3)
            cyc = DistPeriodicLOR(self.mesh, self.lv.p, "helmholtz", self.comm, self.layers,
                                  nu=self.nu, c=c, block=self.block, q1_block=self.q1_block,
                                  levels=self.levels)
            pre = solvers.BlockDiagonalPreconditioner(cyc, 3, self.n)
            self._helm[key] = (op, A, pre)
        return self._helm[key]

    def step(self):
        from .timeint import StepReport, _combo, bdf_coefficients
        k_eff = min(self.k, len(self.u_hist))
        s = bdf_coefficients(k_eff)
        dt, t_new = self.dt, self.t + self.dt
        b0 = s.b[0]
        rep = StepReport(t=t_new)
        nv = 3 * self.n
        terms = [(-s.b[j] / dt, self.u_hist[j - 1]) for j in range(1, k_eff + 1)]
        terms += [(s.a[j - 1], self.n_hist[j - 1]) for j in range(1, k_eff + 1)]
        F = _combo(terms, nv)
        rhs_p = self.Gt.apply(F)
        self.mean.apply_into(rhs_p, rhs_p)
        p, prep = self._cg(self.Lp, rhs_p, self.pressure_pre, 1, x0=self.p, project=self.mean)
        if not prep.converged:
            raise RuntimeError(f"pressure solve failed: {prep}")
        rep.pressure_iters = prep.iterations
        op, A, pre = self._helmholtz(b0)
        b_u = self.M.apply(F)
        vec.axpby(-1.0, self.G.apply(p), 1.0, b_u)
        u, hrep = self._cg(A, b_u, pre, 3)
        if not hrep.converged:
            raise RuntimeError(f"velocity solve failed: {hrep}")
        rep.helmholtz_iters = hrep.iterations
        n_new, it_n = self._nodal_convection(u)
        rep.mass_iters = it_n
        self.u_hist.insert(0, u)
        self.n_hist.insert(0, n_new)
        del self.u_hist[self.k:], self.n_hist[self.k:]
        self.u, self.p, self.t = u, self._weighted_mean_free(p), t_new
        return rep

    def kinetic_energy(self):
        Mu = self.M.apply(self.u)
        e = dev.zeros(1)
        self._dot(self.u, Mu, e, 3)
        return float(e.item()) / (2.0 * self._volume)
