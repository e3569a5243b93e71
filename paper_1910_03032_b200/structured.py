"""Structured-box "scale mode": LOR-preconditioned solves at 100M DoFs.

The reference builds its spaces and LOR hierarchy on the host (numbering:
fespace.py:71-217, ~86 s at 10M DoFs; LOR assembly, interpolation and ILU(0):
lor.py:61-123, solvers.py:269-392, numba_backend.py:64-103, 55-70 s at 1M
DoFs), which cannot reach cfg3's 100M DoFs.  For a structured box
(`cartesian_mesh`, optionally `perturb_mesh`) every piece follows from the
lattice, so this module builds the whole hierarchy on the device
 and runs the scale-mode V-cycle of SURVEY.md 8(e'):

* **Numbering** (`BoxSpace`): block-major first-touch.  DoFs are numbered
  block by block (blocks of `block`^3 elements, x fastest), and inside a block
  in the reference's first-touch order (owner element in scan order, then the
  local lattice index).  Block-Jacobi ILU(0) depends only on the relative
  order inside each block, so the smoother is exactly the one the parity path
  builds from the reference numbering (`solvers.BlockILU0Smoother`), while
  every block's rows are contiguous.  The numbering is closed form per
  lattice point, evaluated with tensor ops on the device.
* **Levels**: the reference's degree ladder p -> ceil(p/2) -> ... -> 1
  (solvers.py:314-318), then, instead of a direct solve of the Q1 level
  (1.6M rows at cfg3 p = 4), geometric coarsening of the Q1 box by 2 per
  direction until the level fits a dense inverse (SURVEY.md 8(e')
  "coarse solve" recommendation).  Q1 levels on coarsened boxes are
  rediscretised on the aggregated cells.
* **Per level** (all on the device): `fb_lor_assemble_box` (CSR),
  `fb_blockilu_create_csr` (block ILU(0) factor + level groups),
  `fb_transfer_*` (matrix-free nodal interpolation, deterministic P^T).

The V-cycle itself is `solvers.LORPreconditioner._cycle` (same V(1,1) order
as solvers.py:375-392).  Only Dirichlet-on-all-boundaries problems (cfg3)
are supported here.
"""

import ctypes as C
import time

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from . import device as dev
from . import geometry
from . import lor as lor_mod
from . import mfop
from . import solvers
from . import vec
from .quadrature import build_eval_matrices, make_basis


DEFAULT_COARSE_CYCLES = 2

# ---------------------------------------------------------------------------
# block-major first-touch numbering of a structured box
# ---------------------------------------------------------------------------

def _axis_tables(n_el, p, block, periodic=False):
    """Per-axis closed-form pieces of the numbering for lattice index g.
    Periodic axes have n_el p lattice points (the last element's local index
    p is the first element's local 0, mesh.py:81-96): the first touch of
    every point is unchanged, the last element owns one point less."""
    N = n_el * p + (0 if periodic else 1)
    g = np.arange(N, dtype=np.int64)
    o = np.maximum(0, (g - 1) // p)             # first-touch owner element
    l = g - o * p                                # local lattice index in the owner
    s = (o > 0).astype(np.int64)                 # first owned local index
    cnt = p + (np.arange(n_el) == 0).astype(np.int64)  # owned lattice points per element
    if periodic:
        cnt[-1] -= 1
    blk = np.arange(n_el) // block
    nb = int(blk[-1]) + 1
    TW = np.bincount(blk, weights=cnt, minlength=nb).astype(np.int64)
    excl = np.cumsum(cnt) - cnt
    SP = excl - excl[blk * block]                # owned points of earlier elements in the block
    return {"N": N, "nb": nb, "TW": TW, "B": blk[o], "C": cnt[o], "SP": SP[o], "R": l - s}


def box_lattice_ids(counts, p, block, device=None, gz_range=None, periodic=(False,) * 3):
    """(Nz, Ny, Nx) int64 tensor: DoF id of every lattice point, plus the
    (nblocks+1) block row offsets (numpy).  gz_range = (g0, g1) restricts the
    result to the lattice planes g0 <= gz < g1 (ids stay global).  Periodic
    axes have counts[a] p lattice points (no duplicated wrap plane)."""
    device = device if device is not None else torch.device("cpu")
    periodic = tuple(bool(v) for v in periodic) if periodic else (False,) * 3
    tx, ty, tz = (_axis_tables(counts[a], p, block, periodic[a]) for a in range(3))
    bsize = (tz["TW"][:, None, None] * ty["TW"][None, :, None] * tx["TW"][None, None, :])
    flat = bsize.ravel()
    block_ptr = np.concatenate([[0], np.cumsum(flat)]).astype(np.int64)
    boff = torch.from_numpy(block_ptr[:-1].reshape(bsize.shape)).to(device)

    def T(a, shape):
        return torch.from_numpy(np.ascontiguousarray(a)).to(device).view(shape)

    if gz_range is not None:
        g0, g1 = gz_range
        tz = {k: (v[g0:g1] if isinstance(v, np.ndarray) and v.shape[0] == tz["N"] else v)
              for k, v in tz.items()}
    zs, ys, xs = (-1, 1, 1), (1, -1, 1), (1, 1, -1)
    Bz, By, Bx = T(tz["B"], zs), T(ty["B"], ys), T(tx["B"], xs)
    TWy, TWx = T(ty["TW"][ty["B"]], ys), T(tx["TW"][tx["B"]], xs)
    ids = boff[Bz, By, Bx]
    ids += T(tz["SP"], zs) * TWy * TWx
    Cz, Cy, Cx = T(tz["C"], zs), T(ty["C"], ys), T(tx["C"], xs)
    ids += Cz * T(ty["SP"], ys) * TWx
    ids += Cz * Cy * T(tx["SP"], xs)
    ids += (T(tz["R"], zs) * Cy + T(ty["R"], ys)) * Cx + T(tx["R"], xs)
    return ids, block_ptr


def lattice_element_dofs(ids, p, periodic=(False,) * 3):
    """(ne, (p+1)^3) element map from the lattice ids (elements x fastest,
    local index i0 + n i1 + n^2 i2).  A periodic axis wraps: its first
    lattice plane is appended before the elements are cut out."""
    n = p + 1
    for a, per in enumerate(periodic or ()):
        if per:
            dim = 2 - a  # ids are (z, y, x)
            ids = torch.cat([ids, ids.narrow(dim, 0, 1)], dim=dim)
    e = ids.unfold(0, n, p).unfold(1, n, p).unfold(2, n, p)
    return e.reshape(-1, n ** 3)


class BoxSpace:
    """Scalar degree-p space on a structured box, numbered block-major.

    Duck-types the attributes of `spaces.FESpace` the operators read
    (`mesh`, `p`, `dim`, `vdim`, `basis`, `element_dofs`, `ndofs_scalar`,
    `boundary_dof_set`)."""

    def __init__(self, mesh, p, block=2, device=None, vdim=1):
        counts = tuple(int(c) for c in mesh.counts)
        if mesh.dim != 3 or len(counts) != 3:
            raise ValueError("BoxSpace needs a structured 3D box mesh")
        self.periodic = tuple(bool(v) for v in (mesh.periodic or (False,) * 3))
        self.mesh = mesh
        self.counts = counts
        self.p = p
        self.block = block
        self.dim = 3
        self.vdim = int(vdim)
        self.basis = make_basis(p)
        self._owner = self._coords = None
        self.device = device if device is not None else torch.device("cpu")
        ids, self.block_ptr = box_lattice_ids(counts, p, block, self.device,
                                              periodic=self.periodic)
        self.ndofs_scalar = int(ids.numel())
        if self.ndofs_scalar >= 2 ** 31:
            raise ValueError("box too large for int32 DoF ids")
        self.lattice_ids = ids.to(torch.int32).contiguous()
        self._ed = None

    @property
    def ndofs(self):
        return self.vdim * self.ndofs_scalar

    @property
    def nloc(self):
        return (self.p + 1) ** 3

    # -- FESpace helpers the callers use (fespace.py:247-340) ------------------
    def _owners(self):
        if self._owner is None:
            flat = self.element_dofs.ravel()
            first = np.full(self.ndofs_scalar, flat.size, dtype=np.int64)
            np.minimum.at(first, flat, np.arange(flat.size))
            self._owner = (first // self.nloc, first % self.nloc)
        return self._owner

    @property
    def dof_owner_elem(self):
        return self._owners()[0]

    @property
    def dof_owner_local(self):
        return self._owners()[1]

    @property
    def node_coords(self):
        """Physical position of every DoF (its first-touch owner element's node)."""
        if self._coords is None:
            from .spaces import element_node_coords
            e, l = self._owners()
            self._coords = element_node_coords(self)[e, l]
        return self._coords

    def expand_dofs(self, scalar_dofs, components=None):
        comps = range(self.vdim) if components is None else components
        ns = self.ndofs_scalar
        return np.concatenate([np.asarray(scalar_dofs) + c * ns for c in comps])

    def project(self, f):
        vals = np.asarray(f(self.node_coords), dtype=np.float64)
        if self.vdim == 1:
            return vals.reshape(-1).copy()
        return vals.T.reshape(-1).copy()

    @property
    def nblocks(self):
        return len(self.block_ptr) - 1

    @property
    def element_dofs(self):
        if self._ed is None:
            ed = lattice_element_dofs(self.lattice_ids, self.p, self.periodic).to(torch.int64)
            self._ed = ed.cpu().numpy()
        return self._ed

    def boundary_dof_set(self, attributes=None):
        if attributes is not None:
            raise ValueError("scale mode constrains the whole boundary")
        L = self.lattice_ids
        px, py, pz = self.periodic
        faces = ([] if pz else [L[0], L[-1]]) + ([] if py else [L[:, 0], L[:, -1]]) + \
                ([] if px else [L[:, :, 0], L[:, :, -1]])
        if not faces:
            return np.zeros(0, dtype=np.int64)
        b = torch.cat([f.reshape(-1) for f in faces]).to(torch.int64)
        return torch.unique(b).cpu().numpy()


# ---------------------------------------------------------------------------
# meshes
# ---------------------------------------------------------------------------

def box_mesh(counts, perturb=0.0, seed=1):
    m = geometry.cartesian_mesh(tuple(counts))
    if perturb:
        m = geometry.perturb_mesh(m, perturb, seed=seed)
    return m


def _coarse_vertex_index(n):
    m = -(-n // 2)
    return np.minimum(2 * np.arange(m + 1), n), m


def can_coarsen_box(mesh):
    """Geometric coarsening applies: at least 2 cells per direction, and
    periodic directions keep >= 3 coarse cells with an even fine count."""
    per = tuple(getattr(mesh, "periodic", ()) or (False,) * 3)
    counts = tuple(mesh.counts)
    if min(counts) < 2:
        return False
    return all(not per[a] or (counts[a] % 2 == 0 and counts[a] // 2 >= 3) for a in range(3))


def coarsen_box(mesh):
    """Box of ceil(n/2) cells per direction whose vertices are every second
    vertex of `mesh` (the last cell spans one fine cell when n is odd).
    Periodic boxes (even counts along periodic axes): coarse cell (I, J, K)
    has the corners of the fine cells (2I + bx, 2J + by, 2K + bz) at its
    corners (bx, by, bz), so the wrap cells keep their physical corners."""
    counts = tuple(mesh.counts)
    per = tuple(getattr(mesh, "periodic", ()) or (False,) * 3)
    if any(per):
        if not can_coarsen_box(mesh):
            raise ValueError("periodic coarsening needs even counts and >= 6 cells per axis")
        mx, my, mz = (c // 2 for c in counts)
        cm = geometry.cartesian_mesh((mx, my, mz), periodic=per)
        Fc = mesh.corners.reshape(counts[2], counts[1], counts[0], 8, 3)
        I, J, K = (np.arange(m) for m in (mx, my, mz))
        corners = np.empty((mz, my, mx, 8, 3))
        for c in range(8):
            bx, by, bz = c & 1, (c >> 1) & 1, (c >> 2) & 1
            corners[:, :, :, c] = Fc[(2 * K + bz)[:, None, None], (2 * J + by)[None, :, None],
                                     (2 * I + bx)[None, None, :], c]
        corners = corners.reshape(-1, 8, 3)
        vertices = np.zeros((cm.num_vertices, 3))
        vertices[cm.elements.ravel()] = corners.reshape(-1, 3)  # identified vertices: one copy
        return geometry.Mesh(3, vertices, cm.elements, corners, cm.boundary_faces, per,
                             (mx, my, mz))
    V = mesh.vertices.reshape(counts[2] + 1, counts[1] + 1, counts[0] + 1, 3)
    (fx, mx), (fy, my), (fz, mz) = (_coarse_vertex_index(n) for n in counts)
    Vc = V[fz][:, fy][:, :, fx].reshape(-1, 3)
    cm = geometry.cartesian_mesh((mx, my, mz))
    return geometry.Mesh(3, Vc, cm.elements, Vc[cm.elements], cm.boundary_faces, cm.periodic,
                         (mx, my, mz))


def h_transfer_tables(n):
    """Per-axis linear interpolation weights of fine element i of an n-cell
    axis inside its parent coarse cell: (tables (3, 2, 2), index (n,), parent (n,))."""
    tables = np.array([[[1.0, 0.0], [0.5, 0.5]],   # even cell of a 2-cell parent
                       [[0.5, 0.5], [0.0, 1.0]],   # odd cell of a 2-cell parent
                       [[1.0, 0.0], [0.0, 1.0]]])  # single-cell parent (odd n)
    i = np.arange(n)
    parent = i // 2
    width = np.minimum(2 * parent + 2, n) - 2 * parent
    idx = np.where(width == 1, 2, i % 2)
    return tables, idx.astype(np.int64), parent


# ---------------------------------------------------------------------------
# device level objects
# ---------------------------------------------------------------------------

class DeviceLevelMatrix(vec.DeviceCSR):
    """LOR matrix of one level, assembled on the device."""

    def __init__(self, space, kind, nu=1.0, c=0.0, constrain=True, pin=None):
        """constrain: Dirichlet rows / columns on the non-periodic box faces
        (lor.py:84-99); pin: one DoF pinned (the pure-Neumann levels,
        solvers.py:361-362)."""
        dev.device()
        corners = torch.from_numpy(np.ascontiguousarray(space.mesh.corners, dtype=np.float64))
        corners = corners.to(dev.device())
        counts = np.asarray(space.counts, dtype=np.int64)
        nodes = np.ascontiguousarray(space.basis.nodes, dtype=np.float64)
        lid = space.lattice_ids.to(dev.device())
        per = getattr(space, "periodic", (False,) * 3)
        faces = 0
        if constrain:
            for a in range(3):
                if not per[a]:
                    faces |= 3 << (2 * a)
        mask = faces | sum((1 << (6 + a)) for a in range(3) if per[a])
        h = C.c_void_p()
        _lib.check(_lib.lib.fb_lor_assemble_box_rows(space.p, _lib.ptr(counts), corners.data_ptr(),
                                                     _lib.ptr(nodes), lid.data_ptr(),
                                                     _lib.KIND[kind], float(nu), float(c), mask,
                                                     -1, -1, C.byref(h)))
        self.handle = h
        if pin is not None:
            _lib.check(_lib.lib.fb_csr_pin(h, int(pin)))
        n = space.ndofs_scalar
        self.shape = (n, n)

    @property
    def nnz(self):
        nnz = C.c_int64(0)
        _lib.check(_lib.lib.fb_csr_info(self.handle, None, None, C.byref(nnz)))
        return int(nnz.value)

    def to_scipy(self):
        n = self.shape[0]
        nnz = self.nnz
        ip = np.empty(n + 1, dtype=np.int64)
        ix = np.empty(max(nnz, 1), dtype=np.int64)
        dv = np.empty(max(nnz, 1), dtype=np.float64)
        _lib.check(_lib.lib.fb_csr_download(self.handle, _lib.ptr(ip), _lib.ptr(ix), _lib.ptr(dv)))
        return sp.csr_matrix((dv[:nnz], ix[:nnz], ip), shape=self.shape)


class DeviceBlockILU0(solvers.BlockILU0Smoother):
    """Block-Jacobi ILU(0) of a block-major device matrix, built on the device."""

    def __init__(self, A, block_ptr):
        self.n = A.shape[0]
        self.jacobi = None
        self._lib = _lib
        bp = np.ascontiguousarray(block_ptr, dtype=np.int64)
        fail = C.c_int64(-1)
        h = C.c_void_p()
        _lib.check(_lib.lib.fb_blockilu_create_csr(A.handle, len(bp) - 1, _lib.ptr(bp),
                                                   C.byref(fail), C.byref(h)))
        if fail.value >= 0:  # zero pivot: damped Jacobi, as solvers.py:283-290
            diag = A.to_scipy().diagonal().copy()
            diag[diag == 0.0] = 1.0
            self.jacobi = 0.6 / diag
            self._jac = dev.to_device(self.jacobi)
            return
        self.handle = h
        self.nblocks = len(bp) - 1


class _Map:
    """Minimal space-like holder for a restriction over an arbitrary map."""

    def __init__(self, dim, p, element_dofs, ndofs):
        self.dim, self.p, self.element_dofs, self.ndofs_scalar = dim, p, element_dofs, ndofs


class BoxTransfer:
    """Nodal interpolation fine <- coarse between two box levels (matrix-free)."""

    def __init__(self, fine, coarse):
        self.fine_r = mfop.restriction(fine)
        if fine.mesh is coarse.mesh:  # p-transfer on the same mesh
            B1, _ = build_eval_matrices(coarse.basis.nodes, fine.basis.nodes)
            W = np.ascontiguousarray(B1, dtype=np.float64)[None]
            widx = np.zeros(sum(fine.counts), dtype=np.int64)
            self.hmap_r = mfop.restriction(coarse)
        else:  # h-transfer: Q1 on the mesh -> Q1 on the coarsened mesh
            if fine.p != 1 or coarse.p != 1:
                raise ValueError("h-transfers connect Q1 levels")
            W = None
            idxs, parents = [], []
            for a in range(3):
                tables, idx, parent = h_transfer_tables(fine.counts[a])
                W = tables
                idxs.append(idx)
                parents.append(parent)
            widx = np.concatenate(idxs)
            mx, my, _ = coarse.counts
            pe = (parents[0][None, None, :] + mx * (parents[1][None, :, None]
                                                   + my * parents[2][:, None, None])).ravel()
            hed = coarse.element_dofs[pe]
            self._hspace = _Map(3, 1, hed, coarse.ndofs_scalar)
            self.hmap_r = mfop.Restriction(self._hspace)
        W = np.ascontiguousarray(W, dtype=np.float64)
        counts = np.asarray(fine.counts, dtype=np.int64)
        h = C.c_void_p()
        _lib.check(_lib.lib.fb_transfer_create(self.fine_r.handle, self.hmap_r.handle,
                                               _lib.ptr(counts), W.shape[0], _lib.ptr(W),
                                               _lib.ptr(widx), C.byref(h)))
        self.handle = h
        per = getattr(fine, "periodic", (False,) * 3)
        if any(per):
            _lib.check(_lib.lib.fb_transfer_set_periodic(
                h, sum(1 << a for a in range(3) if per[a]), *(int(c) for c in fine.counts)))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None and _lib.lib is not None:
            _lib.lib.fb_transfer_destroy(h)

    def prolong_into(self, xc, xf, stream=None):
        _lib.check(_lib.lib.fb_transfer_prolong(self.handle, xc.data_ptr(), xf.data_ptr(),
                                                dev.stream_handle() if stream is None else stream))
        return xf

    def prolong_add_into(self, xc, xf, stream=None):
        """xf += P xc in one pass (bitwise equal to prolong_into + axpby)."""
        _lib.check(_lib.lib.fb_transfer_prolong_add(self.handle, xc.data_ptr(), xf.data_ptr(),
                                                    dev.stream_handle() if stream is None
                                                    else stream))
        return xf

    def restrict_into(self, xf, xc, stream=None):
        _lib.check(_lib.lib.fb_transfer_restrict(self.handle, xf.data_ptr(), xc.data_ptr(),
                                                 dev.stream_handle() if stream is None else stream))
        return xc


class _Prolong:
    def __init__(self, T):
        self.T = T

    def apply_into(self, x, y, stream=None):
        return self.T.prolong_into(x, y, stream)

    def apply_add_into(self, x, y, stream=None):
        return self.T.prolong_add_into(x, y, stream)


class _Restrict:
    def __init__(self, T):
        self.T = T

    def apply_into(self, x, y, stream=None):
        return self.T.restrict_into(x, y, stream)


class BoxLORPreconditioner(solvers.LORPreconditioner):
    """Scale-mode LOR V(1,1) cycle of a structured box, built on the device.

    Same cycle as `solvers.LORPreconditioner` with the block smoother; the
    Q1 level is not solved directly but coarsened geometrically until at most
    `max_coarse` rows remain (dense inverse).  `block` / `q1_block`: element
    cube edge of the smoother blocks on p >= 2 / Q1 levels."""

    def __init__(self, space, kind, nu=1.0, c=0.0, dirichlet_attrs="all", block=2,
                 q1_block=4, max_coarse=20000, coarse_cycles=None, pure_neumann=False):
        """dirichlet_attrs="all": Dirichlet rows on every non-periodic box
        face; None with pure_neumann=True: the periodic / Neumann Poisson
        levels pin DoF 0 and the cycle deflates the mean before and after
        (solvers.py:361-362, 384-390)."""
        if pure_neumann:
            if dirichlet_attrs is not None:
                raise ValueError("pure-Neumann cycle expects no constrained dofs")
        elif dirichlet_attrs != "all":
            raise ValueError("scale mode supports Dirichlet conditions on the whole boundary")
        t0 = time.perf_counter()
        self.pure_neumann = bool(pure_neumann)
        self._proj = solvers.MeanProjector() if pure_neumann else None
        self.smoother_kind = "block"
        ddev = dev.device()
        spaces = [space]
        for deg in lor_mod.degree_ladder(space.p)[1:]:
            spaces.append(BoxSpace(space.mesh, deg, block=block if deg > 1 else q1_block,
                                   device=ddev))
        self.q1_index = len(spaces) - 1  # the ladder's Q1 level on the original mesh
        while spaces[-1].ndofs_scalar > max_coarse and can_coarsen_box(spaces[-1].mesh):
            spaces.append(BoxSpace(coarsen_box(spaces[-1].mesh), 1, block=q1_block, device=ddev))
        self.spaces = spaces
        # near-exact Q1 solve (SURVEY 8(e')): when the Q1 level is coarsened
        # geometrically, the reference's exact SuperLU bottom (solvers.py:372,
        # 376) is replaced by `coarse_cycles` stationary h-multigrid V-cycles
        # on the Q1 hierarchy -- a fixed linear (and symmetric) operator, so
        # the outer CG stays a CG
        if coarse_cycles is None:
            coarse_cycles = DEFAULT_COARSE_CYCLES
        self.coarse_cycles = int(coarse_cycles) if len(spaces) - 1 > self.q1_index else 1
        self._A = [DeviceLevelMatrix(s, kind, nu=nu, c=c, constrain=not pure_neumann,
                                     pin=0 if pure_neumann else None) for s in spaces]
        self.levels = list(zip(spaces, self._A))
        self.smoothers = [DeviceBlockILU0(A, s.block_ptr) for s, A in self.levels[:-1]]
        self.transfers = [BoxTransfer(spaces[i], spaces[i + 1]) for i in range(len(spaces) - 1)]
        self._P = [_Prolong(T) for T in self.transfers]
        self._Pt = [_Restrict(T) for T in self.transfers]
        self._bottom = solvers.DenseInverseSolver(self._A[-1].to_scipy())
        sizes = [s.ndofs_scalar for s in spaces]
        self._x = [dev.empty(n) for n in sizes]
        self._r = [dev.empty(n) for n in sizes]
        self._t = [dev.empty(n) for n in sizes]
        self._t2 = [dev.empty(n) for n in sizes]
        self._rk = self._dk = None
        torch.cuda.synchronize()
        self.setup_seconds = time.perf_counter() - t0

    def _cycle(self, level, r, x, st):
        super()._cycle(level, r, x, st)
        if level != self.q1_index or self.coarse_cycles <= 1:
            return
        A = self._A[level]
        if self._rk is None:
            self._rk, self._dk = dev.empty(r.shape[0]), dev.empty(r.shape[0])
        for _ in range(self.coarse_cycles - 1):  # x += V_h (r - A x)
            A.residual_into(r, x, self._rk, st)
            super()._cycle(level, self._rk, self._dk, st)
            vec.axpby(1.0, self._dk, 1.0, x, st)

    def prepare_multi(self, nv):
        """Workspaces of apply_multi_into for nv components (allocated up front
        so a captured CG loop never allocates)."""
        n0 = self.levels[0][0].ndofs_scalar
        if getattr(self, "_mt", None) is None or self._mt.shape[0] != nv * n0:
            self._mt, self._mt2 = dev.empty(nv * n0), dev.empty(nv * n0)
        return self

    def apply_multi_into(self, r, out, nv, stride, stream=None):
        """nv right-hand sides at a common stride (the components of a vector
        field): every component gets exactly apply_into's V-cycle (bitwise),
        but the fine-level residuals of all components share one pass over the
        level matrix (vec.DeviceCSR.residual_multi_into)."""
        st = dev.stream_handle() if stream is None else stream
        if self.pure_neumann or len(self.levels) < 2 or self.q1_index == 0:
            for c in range(nv):
                self.apply_into(r[c * stride:(c + 1) * stride], out[c * stride:(c + 1) * stride],
                                stream)
            return out
        self.prepare_multi(nv)
        A, sm = self._A[0], self.smoothers[0]
        t, t2 = self._mt, self._mt2
        m = nv * stride

        def sl(v, c):
            return v[c * stride:(c + 1) * stride]

        for c in range(nv):
            sm.forward_into(sl(r, c), sl(out, c), st)
        A.residual_multi_into(nv, stride, r, out, t, st)
        rc, xc = self._r[1], self._x[1]
        for c in range(nv):
            self._Pt[0].apply_into(sl(t, c), rc, st)
            self._cycle(1, rc, xc, st)
            self._P[0].apply_add_into(xc, sl(out, c), st)  # out_c += P xc
        A.residual_multi_into(nv, stride, r, out, t, st)
        if getattr(sm, "adds_in_place", False):
            for c in range(nv):
                sm.backward_add_into(sl(t, c), sl(out, c), st)
        else:
            for c in range(nv):
                sm.backward_into(sl(t, c), sl(t2, c), st)
            vec.axpby(1.0, t2[:m], 1.0, out[:m], st)
        return out

    def clone_workspace(self):
        """Concurrent copy for BlockDiagonalPreconditioner: own level vectors
        and own transfers (a transfer keeps its per-element restriction
        contributions in a device buffer, so clones must not share it)."""
        c = super().clone_workspace()
        if c is not None:
            c._rk = c._dk = None
            c.transfers = [BoxTransfer(self.spaces[i], self.spaces[i + 1])
                           for i in range(len(self.spaces) - 1)]
            c._P = [_Prolong(T) for T in c.transfers]
            c._Pt = [_Restrict(T) for T in c.transfers]
        return c

    def level_bytes(self):
        """Algorithmic HBM bytes of one V-cycle, per level (each datum of the
        cycle's kernels read or written once; CSR / factor entries 12 B = fp64
        value + int32 column, vectors 8 B per row):
          smoother sweep  12 (nnz_L + nnz_U) + 8 n (inverse diagonal) + 16 n (in, out)
          residual        12 nnz(A) + 24 n  (x, r in; t out)
          transfers       8 (n + n_coarse) each way;  axpby 24 n (twice)
        per non-bottom level: 2 sweeps + 2 residuals + both transfers + 2 axpbys;
        the Q1 sub-hierarchy is traversed `coarse_cycles` times (plus one
        residual and one axpby per extra cycle); bottom: dense GEMV 8 nc^2."""
        out = []
        k = self.coarse_cycles
        nl = len(self.levels)
        for i, (sp_, A) in enumerate(self.levels):
            n = sp_.ndofs_scalar
            rep = k if i >= self.q1_index else 1
            if i == nl - 1:
                out.append({"rows": n, "bytes": rep * (8.0 * n * n + 16.0 * n), "kind": "dense"})
                continue
            lo, up = C.c_int64(0), C.c_int64(0)
            sm = self.smoothers[i]
            if getattr(sm, "handle", None) is not None:
                _lib.check(_lib.lib.fb_blockilu_info(sm.handle, None, C.byref(lo), C.byref(up),
                                                     None))
            nnz = A.nnz
            nc = self.spaces[i + 1].ndofs_scalar
            per = (2 * (12.0 * (lo.value + up.value) + 24.0 * n) + 2 * (12.0 * nnz + 24.0 * n)
                   + 2 * 8.0 * (n + nc) + 2 * 24.0 * n)
            extra = (k - 1) * (12.0 * nnz + 24.0 * n + 24.0 * n) if i == self.q1_index else 0.0
            out.append({"rows": n, "nnz_A": nnz, "nnz_ilu": lo.value + up.value,
                        "bytes": rep * per + extra})
        return out

    def describe(self):
        return {"coarse_cycles": self.coarse_cycles, "q1_index": self.q1_index,
                "levels": [{"p": s.p, "counts": list(s.counts), "rows": s.ndofs_scalar,
                            "nnz": A.nnz} for s, A in self.levels]}


def helmholtz_box_problem(counts, p, c=10.0, nu=1.0, perturb=0.05, seed=1, block=2,
                          q1_block=4, max_coarse=20000, rhs_seed=0, coarse_cycles=None):
    """cfg3 building blocks on one device: box mesh, block-major space,
    constrained Helmholtz operator, scale-mode LOR preconditioner and a
    random right-hand side with zero boundary values."""
    t0 = time.perf_counter()
    mesh = box_mesh(counts, perturb=perturb, seed=seed)
    ddev = dev.device()
    space = BoxSpace(mesh, p, block=block, device=ddev)
    geom = geometry.DeviceGeometry(mesh, space.basis.quad)
    op = mfop.HelmholtzOperator(space, geom, c=c, nu=nu)
    bdr = space.boundary_dof_set()
    A = mfop.ConstrainedOperator(op, bdr)
    t1 = time.perf_counter()
    M = BoxLORPreconditioner(space, "helmholtz", nu=nu, c=c, block=block, q1_block=q1_block,
                             max_coarse=max_coarse, coarse_cycles=coarse_cycles)
    g = torch.Generator(device=ddev)
    g.manual_seed(rhs_seed)
    b = torch.randn(space.ndofs_scalar, generator=g, dtype=torch.float64, device=ddev)
    b[torch.from_numpy(bdr).to(ddev)] = 0.0
    torch.cuda.synchronize()
    return {"mesh": mesh, "space": space, "op": op, "A": A, "M": M, "b": b,
            "setup_operator_s": t1 - t0, "setup_precond_s": M.setup_seconds}
