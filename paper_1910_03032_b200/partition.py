"""Element-slab domain decomposition for 1..N GPUs.

The reference has no parallelism; this is the B200 build's multi-GPU layer.
The structured element grid (x-fastest numbering, mesh.py:110-121) is cut into
contiguous z-slabs of whole element layers, so every rank owns a contiguous
element range.  Each rank works on a local space: the DoFs its elements touch,
numbered [owned (global order) | ghosts (global order)], where a DoF is owned
by the rank holding its first-touch owner element (fespace.py:247-263), i.e.
the lowest slab touching it.

* Operator apply: the local fused kernel gives complete values for DoFs
  interior to the slab and partial sums on the cut planes; ``halo_sum`` adds
  the neighbour's partials (lower rank's contribution first on both sides, so
  both copies are bitwise identical).  One send/recv pair per cut per apply,
  ~(p n_cells + 1)^2 doubles.
* Dots: local sum over the owned prefix, then one all-reduce.

Communication goes through ``torch.distributed`` (NCCL between GPUs, gloo in
the CPU tests).  Everything that is not communication stays in libfbb200.
"""

import numpy as np

from .spaces import FESpace


class SlabPartition:
    """Owned/ghost bookkeeping for one rank of a z-slab partition."""

    def __init__(self, space, rank, world, counts=None):
        mesh = space.mesh
        counts = counts or getattr(mesh, "counts", None)
        if not counts:
            from .solvers import infer_counts
            counts = infer_counts(mesh)
        if not counts:
            raise ValueError("slab partitioning needs a structured (x-fastest) element grid")
        self.counts = tuple(counts)
        d = space.dim
        nz = self.counts[-1]
        plane = int(np.prod(self.counts[:-1]))
        if world > nz:
            raise ValueError(f"{world} ranks but only {nz} element layers")
        bounds = np.linspace(0, nz, world + 1).round().astype(int)
        self.layers = (int(bounds[rank]), int(bounds[rank + 1]))
        self.e_lo, self.e_hi = self.layers[0] * plane, self.layers[1] * plane
        self.rank, self.world = rank, world
        self.space = space
        ed = space.element_dofs[self.e_lo:self.e_hi]
        touched = np.unique(ed)
        owner_elem = space.dof_owner_elem[touched]
        owned_mask = (owner_elem >= self.e_lo) & (owner_elem < self.e_hi)
        owned = touched[owned_mask]
        ghosts = touched[~owned_mask]
        self.global_ids = np.concatenate([owned, ghosts])  # local -> global
        self.n_owned = owned.size
        self.n_local = self.global_ids.size
        g2l = {}
        lookup = np.full(space.ndofs_scalar, -1, dtype=np.int64)
        lookup[self.global_ids] = np.arange(self.n_local)
        self._lookup = lookup
        self.local_element_dofs = lookup[ed]
        # shared cut-plane DoFs with each neighbour, in global order
        self.shared = {}
        for nb in (rank - 1, rank + 1):
            if 0 <= nb < world:
                lo = int(bounds[nb]) * plane
                hi = int(bounds[nb + 1]) * plane
                other = np.unique(space.element_dofs[lo:hi])
                common = np.intersect1d(touched, other)
                self.shared[nb] = lookup[common]
        del g2l

    def local_space(self):
        """A space over this rank's elements in local DoF numbering."""
        return LocalSpace(self)

    def scatter_global(self, x_global):
        """Local copy (owned + ghosts) of a global vector (host numpy)."""
        return np.asarray(x_global)[self.global_ids]

    def gather_owned(self, x_local):
        return np.asarray(x_local)[:self.n_owned], self.global_ids[:self.n_owned]


class _LocalMesh:
    def __init__(self, mesh, lo, hi, counts, layers):
        self.dim = mesh.dim
        self.corners = mesh.corners[lo:hi]
        self.elements = mesh.elements[lo:hi]
        self.vertices = mesh.vertices
        self.periodic = getattr(mesh, "periodic", ())
        self.counts = tuple(counts[:-1]) + (layers[1] - layers[0],)
        self.boundary_faces = np.zeros((0, 3), dtype=np.int64)

    @property
    def num_elements(self):
        return self.elements.shape[0]

    @property
    def num_vertices(self):
        return self.vertices.shape[0]


class LocalSpace:
    """FESpace-like view of a slab: what the operators need."""

    def __init__(self, part):
        sp = part.space
        self.partition = part
        self.p = sp.p
        self.dim = sp.dim
        self.vdim = sp.vdim
        self.basis = sp.basis
        self.mesh = _LocalMesh(sp.mesh, part.e_lo, part.e_hi, part.counts, part.layers)
        self.element_dofs = part.local_element_dofs
        self.ndofs_scalar = part.n_local

    @property
    def ndofs(self):
        return self.vdim * self.ndofs_scalar

    @property
    def nloc(self):
        return (self.p + 1) ** self.dim


class HaloExchange:
    """Cut-plane partial-sum exchange over torch.distributed.

    On CUDA tensors the pack/unpack runs as libfbb200 permutation and axpby
    kernels and the transfer is one batched NCCL send/recv per neighbour; on
    CPU tensors (gloo tests) the same steps use torch indexing."""

    def __init__(self, part, device=None):
        import torch
        self.part = part
        self.device = device
        cuda = device is not None and torch.device(device).type == "cuda"
        self.cuda = cuda
        itype = torch.int32 if cuda else torch.long
        self.idx = {nb: torch.as_tensor(np.asarray(ix), dtype=itype, device=device)
                    for nb, ix in part.shared.items()}
        self.sendbuf = {nb: torch.empty(len(ix), dtype=torch.float64, device=device)
                        for nb, ix in part.shared.items()}
        self.recvbuf = {nb: torch.empty(len(ix), dtype=torch.float64, device=device)
                        for nb, ix in part.shared.items()}

    def sum(self, y, comps=1, ns=None):
        """Complete the partial sums of the shared DoFs of y (in place).
        A two-term IEEE sum is commutative, so both neighbours end with
        bitwise identical copies."""
        import torch.distributed as dist
        ns = ns or y.shape[0]
        for c in range(comps):
            yc = y[c * ns:(c + 1) * ns]
            ops = []
            for nb, ix in self.idx.items():
                if self.cuda:
                    from . import vec
                    vec.permute(ix, yc, self.sendbuf[nb], scatter=False)
                else:
                    self.sendbuf[nb].copy_(yc[ix])
                ops.append(dist.P2POp(dist.isend, self.sendbuf[nb], nb))
                ops.append(dist.P2POp(dist.irecv, self.recvbuf[nb], nb))
            if ops:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
            for nb, ix in self.idx.items():
                if self.cuda:
                    from . import vec
                    vec.axpby(1.0, self.recvbuf[nb], 1.0, self.sendbuf[nb])
                    vec.permute(ix, self.sendbuf[nb], yc, scatter=True)
                else:
                    yc[ix] = self.sendbuf[nb] + self.recvbuf[nb]
        return y


class DistributedOperator:
    """y = A x on the slab: local apply + cut-plane halo sum."""

    def __init__(self, local_op, part, halo=None):
        self.op = local_op
        self.part = part
        self.halo = halo or HaloExchange(part, device=None)
        n = local_op.shape[0]
        self.shape = (n, n)

    def apply_into(self, x, y, stream=None):
        self.op.apply_into(x, y)
        vd = getattr(self.op, "space", None)
        comps = vd.vdim if vd is not None else 1
        return self.halo.sum(y, comps=comps, ns=self.part.n_local)


def distributed_dot(x, y, part):
    """Global dot of two local vectors: owned prefix, then all-reduce."""
    import torch
    import torch.distributed as dist
    n = part.n_owned
    s = torch.dot(x[:n], y[:n]).reshape(1) if not x.is_cuda else _device_dot(x[:n], y[:n])
    if dist.is_initialized() and part.world > 1:
        dist.all_reduce(s)
    return s


def _device_dot(x, y):
    from . import vec
    return vec.dot(x, y)


class StructuredSlab:
    """One rank's z-slab of a global structured box, built locally.

    For weak-scaling runs no rank materialises the global mesh: rank r builds
    the cartesian mesh of layers [r*nz, (r+1)*nz) of a box with `world*nz`
    layers, perturbs only vertices off the cut planes (cut planes stay
    planar, like the domain boundary in perturb_mesh), and numbers it with
    the reference numbering.  The DoFs of the bottom/top cut plane are listed
    in plane-lattice order, which both neighbours compute identically, so the
    halo exchange needs no global ids.
    """

    def __init__(self, counts_xy, nz, p, rank, world, perturb=0.05, seed=1):
        from . import geometry
        d = len(counts_xy) + 1
        self.rank, self.world = rank, world
        z0, z1 = rank * nz / (world * nz), (rank + 1) * nz / (world * nz)
        counts = tuple(counts_xy) + (nz,)
        lows = (0.0,) * (d - 1) + (z0,)
        highs = (1.0,) * (d - 1) + (z1,)
        m = geometry.cartesian_mesh(counts, lows=lows, highs=highs)
        if perturb:
            m = geometry.perturb_mesh(m, perturb, seed=seed + rank)
        self.mesh = m
        self.space = FESpace(m, p)
        self.p = p
        ne_plane = int(np.prod(counts_xy))
        n = p + 1
        ed = self.space.element_dofs
        lat = np.indices((n,) * d).reshape(d, -1)[::-1]  # lat[a] per local index
        cells = np.indices(tuple(counts_xy)[::-1]).reshape(d - 1, -1)[::-1]
        self.planes = {}
        for side, layer, kk in (("bottom", 0, 0), ("top", nz - 1, p)):
            elems = np.arange(layer * ne_plane, (layer + 1) * ne_plane)
            sel = np.flatnonzero(lat[d - 1] == kk)
            dofs = ed[elems][:, sel]  # (ne_plane, n^(d-1))
            # global plane-lattice position of each entry
            key = np.zeros(dofs.shape, dtype=np.int64)
            stride = 1
            for a in range(d - 1):
                pos = cells[a][:, None] * p + lat[a][sel][None, :]
                key += pos * stride
                stride *= counts_xy[a] * p + 1
            uk, first = np.unique(key.ravel(), return_index=True)
            self.planes[side] = dofs.ravel()[first]
        self.shared = {}
        if rank > 0:
            self.shared[rank - 1] = self.planes["bottom"]
        if rank + 1 < world:
            self.shared[rank + 1] = self.planes["top"]
        # owned = everything except the bottom plane (owned by the rank below)
        owned = np.ones(self.space.ndofs_scalar, dtype=bool)
        if rank > 0:
            owned[self.planes["bottom"]] = False
        self.owned_mask = owned
        self.n_local = self.space.ndofs_scalar
