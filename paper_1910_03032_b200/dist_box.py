"""Multi-GPU scale mode: the cfg3 LOR-PCG solve sharded over z-slabs.

SURVEY.md 8(e): the operator, the Krylov vectors and the block-Jacobi ILU(0)
V-cycle shard over element z-slabs with neighbour exchanges only; the Q1
coarse problem is agglomerated.  The block-major numbering of
`structured.BoxSpace` makes this cheap: a slab of whole smoother blocks owns
a CONTIGUOUS range of global DoF ids, so rank r's owned vector is the slice
[off_r, off_{r+1}) of the global vector and the global solution is the
concatenation of the ranks' owned parts.

Per rank and level, local vectors are [owned | bottom ghost plane | top+1
ghost plane] (ghost planes in plane-lattice order, so neighbour messages are
dense plane arrays):

* operator apply (matrix-free, rank's elements only): update the bottom ghost
  plane, apply, send the bottom plane's partial sums down and add the partial
  sums received from above into the owned top plane;
* LOR level matrices: owned rows assembled completely on the device
  (`fb_lor_assemble_box_rows` over the slab plus one element layer above),
  columns owned + both ghost planes; SpMV after a two-plane ghost update;
* block-Jacobi ILU(0): the rank's blocks only -- identical math to one GPU;
* transfers: prolongation writes owned fine DoFs from the rank's elements
  (coarse ghosts updated first), restriction sums element contributions and
  exchanges the cut-plane partial sums like the operator;
* Q1 coarse problem: owned parts all-gathered (13 MB at cfg3 p = 4) and the
  whole Q1 V-cycle (geometric coarsening + dense bottom) run redundantly on
  every rank;
* dots: owned slice + all-reduce.

`Comm` has two implementations: `TorchComm` (torch.distributed: NCCL between
GPUs, one process per GPU) and `ThreadComm`, which runs R ranks as threads of
one process on one GPU with host-side barriers only (no kernel ever waits on
another rank's kernel), used to test the sharded path on a single device.
"""

import ctypes as C
import threading

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
from .quadrature import build_eval_matrices, make_basis


# ---------------------------------------------------------------------------
# communication
# ---------------------------------------------------------------------------

class TorchComm:
    """torch.distributed communicator (NCCL on GPUs)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()

    def exchange(self, send_down, send_up, recv_down, recv_up):
        """Send to rank-1 / rank+1 and receive from them (None: no message)."""
        ops = []
        P2P = self.dist.P2POp
        if send_down is not None:
            ops.append(P2P(self.dist.isend, send_down, self.rank - 1))
        if recv_down is not None:
            ops.append(P2P(self.dist.irecv, recv_down, self.rank - 1))
        if send_up is not None:
            ops.append(P2P(self.dist.isend, send_up, self.rank + 1))
        if recv_up is not None:
            ops.append(P2P(self.dist.irecv, recv_up, self.rank + 1))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()

    def exchange_ring(self, send_down, send_up, recv_down, recv_up):
        """Periodic neighbours (rank -+ 1 mod world), in two phases (all
        up-going messages, then all down-going ones) so that a 2-rank ring,
        where both neighbours are the same peer, pairs messages correctly."""
        w = self.world
        up, down = (self.rank + 1) % w, (self.rank - 1) % w
        P2P = self.dist.P2POp
        for ops in ([(send_up, self.dist.isend, up), (recv_down, self.dist.irecv, down)],
                    [(send_down, self.dist.isend, down), (recv_up, self.dist.irecv, up)]):
            ops = [P2P(fn, t, peer) for t, fn, peer in ops if t is not None]
            if ops:
                for req in self.dist.batch_isend_irecv(ops):
                    req.wait()

    def allreduce_sum(self, t):
        self.dist.all_reduce(t)
        return t

    def barrier(self):
        self.dist.barrier()

    def allgather(self, t, sizes):
        """Concatenation of every rank's t[:sizes[rank]] (ranks in order)."""
        m = max(sizes)
        buf = torch.zeros(m, dtype=t.dtype, device=t.device)
        buf[:t.shape[0]] = t
        out = torch.empty(m * self.world, dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, buf)
        return torch.cat([out[r * m:r * m + sizes[r]] for r in range(self.world)])


class ThreadHub:
    """Shared state of R in-process ranks (one thread each, one GPU).  A
    baton lock lets exactly one rank thread run host code (and enqueue device
    work) at a time; it is released only while a rank waits at a barrier, so
    ranks run one after another between communication points -- the
    multi-process semantics without concurrent host threads in torch / the C
    library."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.baton = threading.Lock()
        self.slots = {}


class ThreadComm:
    """In-process emulation of the slab exchanges: every rank is a thread on
    the same device; a message is a device tensor handed over at a host
    barrier after torch.cuda.synchronize(), so no kernel waits on another."""

    def __init__(self, hub, rank):
        self.hub = hub
        self.rank = rank
        self.world = hub.world

    def _sync(self):
        try:
            torch.cuda.synchronize()
        except BaseException:
            self.hub.barrier.abort()
            raise
        self.hub.baton.release()
        try:
            self.hub.barrier.wait()
        finally:
            self.hub.baton.acquire()

    def exchange(self, send_down, send_up, recv_down, recv_up):
        h, r = self.hub, self.rank
        h.slots[(r, "down")] = send_down
        h.slots[(r, "up")] = send_up
        self._sync()
        if recv_down is not None:
            recv_down.copy_(h.slots[(r - 1, "up")])
        if recv_up is not None:
            recv_up.copy_(h.slots[(r + 1, "down")])
        self._sync()

    def exchange_ring(self, send_down, send_up, recv_down, recv_up):
        h, r, w = self.hub, self.rank, self.world
        h.slots[(r, "rdown")] = send_down
        h.slots[(r, "rup")] = send_up
        self._sync()
        if recv_down is not None:
            recv_down.copy_(h.slots[((r - 1) % w, "rup")])
        if recv_up is not None:
            recv_up.copy_(h.slots[((r + 1) % w, "rdown")])
        self._sync()

    def barrier(self):
        self._sync()

    def allreduce_sum(self, t):
        h, r = self.hub, self.rank
        h.slots[(r, "red")] = t.clone()
        self._sync()
        acc = h.slots[(0, "red")].clone()
        for q in range(1, self.world):  # fixed rank order: identical on all ranks
            acc += h.slots[(q, "red")]
        self._sync()
        t.copy_(acc)
        return t

    def allgather(self, t, sizes):
        h, r = self.hub, self.rank
        h.slots[(r, "gat")] = t[:sizes[r]].clone()
        self._sync()
        out = torch.cat([h.slots[(q, "gat")] for q in range(self.world)])
        self._sync()
        return out


def run_threads(world, fn):
    """Run fn(comm) for ranks 0..world-1 as threads on the current device;
    returns the per-rank results (re-raises the first exception)."""
    if torch.cuda.is_available():
        # lazy CUDA / cuSOLVER initialisation must not race between the rank threads
        torch.cuda.init()
        torch.linalg.inv(torch.eye(2, dtype=torch.float64, device=dev.device()))
    hub = ThreadHub(world)
    res, err = [None] * world, [None]

    def body(r):
        hub.baton.acquire()
        try:
            res[r] = fn(ThreadComm(hub, r))
        except BaseException as e:  # noqa: BLE001 -- surfaced below
            err[0] = err[0] or e
            hub.barrier.abort()
        finally:
            try:
                if torch.cuda.is_available():
                    torch.cuda.synchronize()
            except BaseException as e:  # noqa: BLE001 -- a device fault: surfaced below
                err[0] = err[0] or e
            hub.baton.release()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err[0] is not None:
        raise err[0]
    return res


# ---------------------------------------------------------------------------
# slab layout of one level
# ---------------------------------------------------------------------------

def slab_layers(nz, world, unit):
    """Element-layer bounds per rank, in whole units of `unit` layers."""
    if nz % unit:
        raise ValueError(f"nz={nz} must be a multiple of the slab unit {unit}")
    nu = nz // unit
    if nu < world:
        raise ValueError(f"{world} ranks but only {nu} slab units")
    b = (np.arange(world + 1) * nu) // world
    return [(int(b[r]) * unit, int(b[r + 1]) * unit) for r in range(world)]


class SlabLevel:
    """Rank r's view of one level (degree p, smoother blocks of `block`
    elements) of a global box partitioned into z-slabs."""

    def __init__(self, mesh, p, block, layers, rank, world, device):
        self.gmesh, self.p, self.block = mesh, p, block
        self.rank, self.world = rank, world
        nx, ny, nz = (int(c) for c in mesh.counts)
        self.counts = (nx, ny, nz)
        e0, e1 = layers[rank]
        if e0 % block or e1 % block:
            raise ValueError("slab bounds must align with smoother blocks")
        self.e0, self.e1 = e0, e1
        self.down, self.up = rank > 0, rank < world - 1
        Nx, Ny = nx * p + 1, ny * p + 1
        self.P = Nx * Ny
        nbx, nby = -(-nx // block), -(-ny // block)
        # owned global range = the rank's blocks (block-major numbering)
        _, bptr = S.box_lattice_ids((nx, ny, nz), p, block, torch.device("cpu"), gz_range=(0, 1))
        b0, b1 = (e0 // block) * nby * nbx, (e1 // block) * nby * nbx
        self.off, self.n_own = int(bptr[b0]), int(bptr[b1] - bptr[b0])
        self.block_ptr = bptr[b0:b1 + 1] - bptr[b0]
        self.ghost_down = self.n_own if self.down else None
        self.ghost_up = self.n_own + (self.P if self.down else 0) if self.up else None
        self.n_local = self.n_own + self.P * (int(self.down) + int(self.up))
        # global ids of the lattice planes [e0 p, (e1 + up) p] (+1 extra: the LOR rows
        # of the top plane need the element layer above)
        gz0, gz1 = e0 * p, min(e1 + (1 if self.up else 0), nz) * p + 1
        gids, _ = S.box_lattice_ids((nx, ny, nz), p, block, device, gz_range=(gz0, gz1))
        loc = gids - self.off
        own = (loc >= 0) & (loc < self.n_own)
        plane = torch.arange(self.P, device=device, dtype=torch.int64).view(Ny, Nx)
        gz = torch.arange(gz0, gz1, device=device).view(-1, 1, 1)
        lidx = torch.full_like(loc, -1)
        lidx = torch.where(own, loc, lidx)
        if self.down:
            lidx = torch.where((gz == e0 * p) & ~own, self.ghost_down + plane, lidx)
        if self.up:
            lidx = torch.where((gz == e1 * p + 1) & ~own, self.ghost_up + plane, lidx)
        # local lattice of the rank's elements (operator / transfers)
        self.lid_elems = lidx[: (e1 - e0) * p + 1].to(torch.int32).contiguous()
        self.lid_ext = lidx.to(torch.int32).contiguous()  # + layer above (LOR rows)
        if int((self.lid_elems < 0).sum()) != 0:
            raise RuntimeError("unmapped lattice point in the slab")
        # plane index maps (plane-lattice order)
        top = lidx[(e1 - e0) * p].reshape(-1)
        self.top_plane = top.to(torch.int32).contiguous()          # owned, gz = e1 p
        self.bot_plus1 = lidx[1].reshape(-1).to(torch.int32).contiguous()  # owned, gz = e0 p + 1
        self.bot_plane = lidx[0].reshape(-1).to(torch.int32).contiguous()  # gz = e0 p
        self.device = device
        # rank-local mesh of the slab elements (and one layer above)
        self.mesh_elems = _sub_mesh(mesh, e0, e1)
        self.mesh_ext = _sub_mesh(mesh, e0, min(e1 + (1 if self.up else 0), nz))
        self.mesh = self.mesh_elems  # what the operator / restriction see
        self.basis = make_basis(p)
        self.dim, self.vdim = 3, 1
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
            ed = S.lattice_element_dofs(self.lid_elems, self.p).to(torch.int64)
            self._buf["ed"] = ed.cpu().numpy()
        return self._buf["ed"]

    def boundary_local(self):
        """Local ids (owned and ghost) of global-boundary lattice points."""
        L = self.lid_ext
        nx, ny, nz = self.counts
        faces = [L[:, 0], L[:, -1], L[:, :, 0], L[:, :, -1]]
        if self.rank == 0:
            faces.append(L[0])
        if not self.up:
            faces.append(L[-1])
        b = torch.cat([f.reshape(-1) for f in faces]).to(torch.int64)
        b = b[b >= 0]
        return torch.unique(b).cpu().numpy()

    def buf(self, name, n):
        t = self._buf.get(name)
        if t is None or t.shape[0] != n:
            t = self._buf[name] = torch.empty(n, dtype=torch.float64, device=self.device)
        return t

    # -- halo operations -----------------------------------------------------------
    def ghost_update(self, comm, x, top1=True):
        """Fill the ghost planes of x from the owners: bottom plane from rank-1
        (its owned top plane), top+1 plane from rank+1 (its owned bottom+1)."""
        P = self.P
        send_up = self.buf("su", P) if self.up else None
        send_down = self.buf("sd", P) if (self.down and top1) else None
        if send_up is not None:
            vec.permute(self.top_plane, x, send_up)
        if send_down is not None:
            vec.permute(self.bot_plus1, x, send_down)
        recv_down = x[self.ghost_down:self.ghost_down + P] if self.down else None
        recv_up = x[self.ghost_up:self.ghost_up + P] if (self.up and top1) else None
        comm.exchange(send_down, send_up, recv_down, recv_up)

    def sum_planes(self, comm, y):
        """Cut-plane partial sums: send the bottom ghost plane's partials down,
        add the partials received from above into the owned top plane."""
        P = self.P
        send_down = y[self.ghost_down:self.ghost_down + P] if self.down else None
        recv_up = self.buf("ru", P) if self.up else None
        comm.exchange(send_down, None, None, recv_up)
        if recv_up is not None:
            _lib.check(_lib.lib.fb_index_add(P, self.top_plane.data_ptr(), recv_up.data_ptr(),
                                             y.data_ptr(), dev.stream_handle()))


def _sub_mesh(mesh, e0, e1):
    nx, ny, nz = mesh.counts
    plane = nx * ny
    corners = mesh.corners[e0 * plane:e1 * plane]
    cm = geometry.cartesian_mesh((nx, ny, e1 - e0))  # local connectivity (unused by the kernels)
    return geometry.Mesh(3, cm.vertices, cm.elements, corners, cm.boundary_faces, cm.periodic,
                         (nx, ny, e1 - e0))


# ---------------------------------------------------------------------------
# distributed pieces
# ---------------------------------------------------------------------------

class DistOperator:
    """Matrix-free operator on the rank's elements + cut-plane partial sums."""

    def __init__(self, op_local, level, comm):
        self.op, self.level, self.comm = op_local, level, comm
        self.shape = (level.n_local, level.n_local)

    def apply_into(self, x, y, stream=None):
        lv = self.level
        lv.ghost_update(self.comm, x, top1=False)
        self.op.apply_into(x, y, stream)
        lv.sum_planes(self.comm, y)
        return y


class DistLevelMatrix(vec.DeviceCSR):
    """Owned rows of a level's LOR matrix (complete), columns owned + ghosts."""

    def __init__(self, level, kind, nu, c, constrain):
        lv = level
        corners = torch.from_numpy(np.ascontiguousarray(lv.mesh_ext.corners, dtype=np.float64))
        corners = corners.to(dev.device())
        counts = np.asarray(lv.mesh_ext.counts, dtype=np.int64)
        nodes = np.ascontiguousarray(lv.basis.nodes, dtype=np.float64)
        faces = 0
        if constrain:
            faces = 1 | 2 | 4 | 8 | (16 if lv.rank == 0 else 0) | (32 if not lv.up else 0)
        h = C.c_void_p()
        _lib.check(_lib.lib.fb_lor_assemble_box_rows(
            lv.p, _lib.ptr(counts), corners.data_ptr(), _lib.ptr(nodes), lv.lid_ext.data_ptr(),
            _lib.KIND[kind], float(nu), float(c), faces, lv.n_own, lv.n_local, C.byref(h)))
        self.handle = h
        self.shape = (lv.n_own, lv.n_local)


class DistTransfer(S.BoxTransfer):
    """p-transfer between two slab levels of the same mesh slab."""

    def __init__(self, fine, coarse):
        self.fine_r = mfop.restriction(fine)
        self.hmap_r = mfop.restriction(coarse)
        B1, _ = build_eval_matrices(coarse.basis.nodes, fine.basis.nodes)
        W = np.ascontiguousarray(B1, dtype=np.float64)[None]
        nx, ny, _ = fine.counts
        counts = np.asarray([nx, ny, fine.e1 - fine.e0], dtype=np.int64)
        widx = np.zeros(int(counts.sum()), dtype=np.int64)
        h = C.c_void_p()
        _lib.check(_lib.lib.fb_transfer_create(self.fine_r.handle, self.hmap_r.handle,
                                               _lib.ptr(counts), 1, _lib.ptr(W), _lib.ptr(widx),
                                               C.byref(h)))
        self.handle = h
        _lib.check(_lib.lib.fb_transfer_set_origin(h, 0, 0, fine.e0))


class DistHTransfer(S.BoxTransfer):
    """h-transfer from a rank's Q1 slab to the whole (agglomerated) coarsened
    Q1 box: the slab's fine elements with their parents' global coarse DoFs.
    Restriction gives this slab's partial coarse vector (summed over ranks by
    the caller); prolongation writes the slab's owned fine DoFs."""

    def __init__(self, fine, coarse):
        self.fine_r = mfop.restriction(fine)
        nx, ny, nz = fine.counts
        W, ix, px = S.h_transfer_tables(nx)
        _, iy, py = S.h_transfer_tables(ny)
        _, iz, pz = S.h_transfer_tables(nz)
        iz, pz = iz[fine.e0:fine.e1], pz[fine.e0:fine.e1]
        widx = np.concatenate([ix, iy, iz])
        mx, my, _ = coarse.counts
        pe = (px[None, None, :] + mx * (py[None, :, None] + my * pz[:, None, None])).ravel()
        self._hspace = S._Map(3, 1, coarse.element_dofs[pe], coarse.ndofs_scalar)
        self.hmap_r = mfop.Restriction(self._hspace)
        W = np.ascontiguousarray(W, dtype=np.float64)
        counts = np.asarray([nx, ny, fine.e1 - fine.e0], dtype=np.int64)
        h = C.c_void_p()
        _lib.check(_lib.lib.fb_transfer_create(self.fine_r.handle, self.hmap_r.handle,
                                               _lib.ptr(counts), W.shape[0], _lib.ptr(W),
                                               _lib.ptr(widx), C.byref(h)))
        self.handle = h
        _lib.check(_lib.lib.fb_transfer_set_origin(h, 0, 0, fine.e0))


class DistLORPreconditioner:
    """Sharded scale-mode V(1,1) cycle (same recursion as
    solvers.LORPreconditioner._cycle, solvers.py:375-392), levels p >= 2 on
    the slabs.  Q1 level: when the single-GPU hierarchy coarsens it
    geometrically (more than max_coarse rows), the Q1 level itself is sharded
    too -- its `coarse_cycles` stationary cycles run on the slabs, and only
    the h-coarsened levels (1/8 of the Q1 rows and below) are agglomerated
    (one all-reduce of the restricted residual per cycle) and solved
    redundantly; otherwise the whole Q1 problem is agglomerated."""

    def __init__(self, mesh, p, kind, comm, layers, nu=1.0, c=0.0, block=2, q1_block=4,
                 max_coarse=20000, levels=None, distribute_q1=True, coarse_cycles=None):
        self.comm = comm
        r, w = comm.rank, comm.world
        ddev = dev.device()
        degs = [d for d in lor_mod.degree_ladder(p) if d > 1]
        self.levels = levels or [SlabLevel(mesh, d, block, layers, r, w, ddev) for d in degs]
        self.q1 = SlabLevel(mesh, 1, q1_block, layers, r, w, ddev)
        self._A = [DistLevelMatrix(lv, kind, nu, c, True) for lv in self.levels]
        self.smoothers = [S.DeviceBlockILU0(A, lv.block_ptr) for A, lv in zip(self._A, self.levels)]
        chain = self.levels + [self.q1]
        self.transfers = [DistTransfer(chain[i], chain[i + 1]) for i in range(len(self.levels))]
        q1_rows = int(np.prod([a + 1 for a in mesh.counts]))
        self.q1_sharded = bool(distribute_q1 and q1_rows > max_coarse
                               and min(mesh.counts) >= 2)
        if self.q1_sharded:
            # sharded Q1 level; h-coarsened hierarchy agglomerated (one V-cycle each)
            self.coarse_cycles = int(coarse_cycles if coarse_cycles is not None
                                     else S.DEFAULT_COARSE_CYCLES)
            self._Aq = DistLevelMatrix(self.q1, kind, nu, c, True)
            self.smq = S.DeviceBlockILU0(self._Aq, self.q1.block_ptr)
            hspace = S.BoxSpace(S.coarsen_box(mesh), 1, block=q1_block, device=ddev)
            self.hT = DistHTransfer(self.q1, hspace)
            self.coarse = S.BoxLORPreconditioner(hspace, kind, nu=nu, c=c, q1_block=q1_block,
                                                 max_coarse=max_coarse, coarse_cycles=1)
            nh = hspace.ndofs_scalar
            self._rh, self._xh = dev.zeros(nh), dev.zeros(nh)
            nq = self.q1.n_local
            self._rk, self._dk = dev.zeros(nq), dev.zeros(nq)
        else:
            # agglomerated Q1 problem: the whole Q1 V-cycle on every rank
            q1space = S.BoxSpace(mesh, 1, block=q1_block, device=ddev)
            self.coarse = S.BoxLORPreconditioner(q1space, kind, nu=nu, c=c, q1_block=q1_block,
                                                 max_coarse=max_coarse)
        sizes = torch.tensor([self.q1.n_own], dtype=torch.float64, device=ddev)
        allsz = comm.allgather(sizes, [1] * w)
        self.q1_sizes = [int(v) for v in allsz.tolist()]
        self.q1_offsets = np.concatenate([[0], np.cumsum(self.q1_sizes)]).astype(np.int64)
        self._x = [dev.zeros(lv.n_local) for lv in chain]
        self._r = [dev.zeros(lv.n_local) for lv in chain]
        self._t = [dev.zeros(lv.n_local) for lv in chain]
        self._t2 = [dev.zeros(lv.n_local) for lv in chain]
        self._q1_ghost_ids = None

    def _q1_vcycle(self, r, x):
        """One V-cycle from the sharded Q1 level: slab block-ILU smoothing and
        residuals, restriction to the agglomerated h-coarse box (partial
        vectors summed over ranks), its V-cycle on every rank, prolongation
        back to the owned fine DoFs (structured.BoxLORPreconditioner._cycle
        at the Q1 level, solvers.py:375-392)."""
        q1, A, sm = self.q1, self._Aq, self.smq
        n = q1.n_own
        t, t2 = self._t[-1], self._t2[-1]
        sm.forward_into(r, x)
        q1.ghost_update(self.comm, x)
        A.residual_into(r, x, t)
        self.hT.restrict_into(t, self._rh)
        self.comm.allreduce_sum(self._rh)
        self.coarse.apply_into(self._rh, self._xh)
        self.hT.prolong_add_into(self._xh, x)  # owned x += P xc; ghosts refreshed below
        q1.ghost_update(self.comm, x)
        A.residual_into(r, x, t)
        sm.backward_into(t, t2)
        vec.axpby(1.0, t2[:n], 1.0, x[:n])

    def _coarse_solve(self, rq, xq):
        """rq: Q1 slab vector with owned residual; xq <- owned correction +
        bottom ghost plane (what the prolongation reads)."""
        q1 = self.q1
        if self.q1_sharded:
            # coarse_cycles stationary cycles: x = V r; x += V (r - A x)
            self._q1_vcycle(rq, xq)
            for _ in range(self.coarse_cycles - 1):
                q1.ghost_update(self.comm, xq)
                self._Aq.residual_into(rq, xq, self._rk)
                self._q1_vcycle(self._rk, self._dk)
                vec.axpby(1.0, self._dk[:q1.n_own], 1.0, xq[:q1.n_own])
            q1.ghost_update(self.comm, xq, top1=False)
            return
        rg = self.comm.allgather(rq[:q1.n_own], self.q1_sizes)
        xg = torch.empty_like(rg)
        self.coarse.apply_into(rg, xg)
        o = int(self.q1_offsets[self.comm.rank])
        vec.copy(xg[o:o + q1.n_own], xq[:q1.n_own])
        if q1.down:
            if self._q1_ghost_ids is None:
                # global Q1 ids of the bottom ghost plane (owned by rank-1)
                gids, _ = S.box_lattice_ids(q1.counts, 1, q1.block, dev.device(),
                                            gz_range=(q1.e0, q1.e0 + 1))
                self._q1_ghost_ids = gids.reshape(-1).to(torch.int32).contiguous()
            vec.permute(self._q1_ghost_ids, xg, xq[q1.ghost_down:q1.ghost_down + q1.P])

    def _cycle(self, i, r, x):
        lv, A, sm = self.levels[i], self._A[i], self.smoothers[i]
        n = lv.n_own
        t, t2 = self._t[i], self._t2[i]
        sm.forward_into(r, x)
        lv.ghost_update(self.comm, x)
        A.residual_into(r, x, t)
        rc, xc = self._r[i + 1], self._x[i + 1]
        T = self.transfers[i]
        T.restrict_into(t, rc)
        cl = self.levels[i + 1] if i + 1 < len(self.levels) else self.q1
        cl.sum_planes(self.comm, rc)
        if i + 1 < len(self.levels):
            self._cycle(i + 1, rc, xc)
            cl.ghost_update(self.comm, xc, top1=False)
        else:
            self._coarse_solve(rc, xc)
        T.prolong_add_into(xc, x)  # owned x += P xc; ghosts refreshed below
        lv.ghost_update(self.comm, x)
        A.residual_into(r, x, t)
        sm.backward_into(t, t2)
        vec.axpby(1.0, t2[:n], 1.0, x[:n])

    def apply_into(self, r, out, stream=None):
        self._cycle(0, r, out)
        return out


def dist_cg(A, b, M, comm, n_own, config=None):
    """solvers.cg with owned-slice dots + all-reduce."""

    def inner(x, y, out):
        vec.dot_into(x[:n_own], y[:n_own], out)
        comm.allreduce_sum(out)
        return out

    return solvers.cg(A, b, precond=M, config=config, inner=inner)


def helmholtz_slab_problem(comm, counts, p, c=10.0, nu=1.0, perturb=0.05, seed=1, block=2,
                           q1_block=4, max_coarse=20000, rhs_seed=0, mesh=None,
                           distribute_q1=True):
    """One rank's share of the cfg3 problem: slab operator (constrained),
    sharded LOR V-cycle, owned part of the global random right-hand side."""
    r, w = comm.rank, comm.world
    ddev = dev.device()
    mesh = mesh if mesh is not None else S.box_mesh(counts, perturb=perturb, seed=seed)
    unit = int(np.lcm(block, q1_block))
    layers = slab_layers(counts[2], w, unit)
    degs = [d for d in lor_mod.degree_ladder(p) if d > 1]
    levels = [SlabLevel(mesh, d, block, layers, r, w, ddev) for d in degs]
    lv = levels[0]
    geom = geometry.DeviceGeometry(lv.mesh_elems, lv.basis.quad)
    op_local = mfop.HelmholtzOperator(lv, geom, c=c, nu=nu)
    bdr = lv.boundary_local()
    A = mfop.ConstrainedOperator(DistOperator(op_local, lv, comm), bdr)
    M = DistLORPreconditioner(mesh, p, "helmholtz", comm, layers, nu=nu, c=c, block=block,
                              q1_block=q1_block, max_coarse=max_coarse, levels=levels,
                              distribute_q1=distribute_q1)
    # global right-hand side, generated identically everywhere; owned slice kept
    N = int(np.prod([counts[a] * p + 1 for a in range(3)]))
    g = torch.Generator(device=ddev)
    g.manual_seed(rhs_seed)
    bg = torch.randn(N, generator=g, dtype=torch.float64, device=ddev)
    b = dev.zeros(lv.n_local)
    vec.copy(bg[lv.off:lv.off + lv.n_own], b[:lv.n_own])
    b[torch.from_numpy(bdr).to(ddev)] = 0.0
    return {"level": lv, "A": A, "M": M, "b": b, "layers": layers, "mesh": mesh}
