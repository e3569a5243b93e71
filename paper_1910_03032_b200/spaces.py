"""Continuous nodal spaces on tensor-product meshes (host-side setup).

``FESpace`` exposes the attributes the reference's operators and solvers
read (fespace.py:31-391): ``element_dofs`` (the L->E map), ``ndofs_scalar``,
``vdim``, ``basis``, boundary DoF sets and DoF owners.  The numbering is the
reference's (vertices, edge interiors, face interiors, element interiors,
each in order of first appearance), computed by the C++ routine
``fb_number_dofs_host`` instead of a per-element Python loop, so reference
spaces and these spaces are interchangeable.
"""

import ctypes as C

import numpy as np

from . import _lib
from .quadrature import make_basis


def local_lattice(p, d):
    n = p + 1
    idx = np.arange(n ** d)
    return np.stack([(idx // n ** a) % n for a in range(d)], axis=1)


def number_dofs(mesh, p):
    """(element_dofs, ndofs_scalar, num_edges, num_faces) via the C++ numbering."""
    d = mesh.dim
    elems = np.ascontiguousarray(mesh.elements, dtype=np.int64)
    ne = elems.shape[0]
    out = np.empty((ne, (p + 1) ** d), dtype=np.int64)
    n_edges = C.c_int64(0)
    n_faces = C.c_int64(0)
    nd = _lib.lib.fb_number_dofs_host(d, p, ne, mesh.num_vertices, _lib.ptr(elems), _lib.ptr(out),
                                      C.byref(n_edges), C.byref(n_faces))
    if nd < 0:
        _lib.check(int(-nd))
    return out, int(nd), int(n_edges.value), int(n_faces.value)


def element_node_coords(space):
    """(ne, nloc, d) physical nodal lattice positions per element."""
    d = space.dim
    t = space.basis.nodes[local_lattice(space.p, d)]  # (nloc, d)
    shp = np.ones((t.shape[0], 2 ** d))
    for c in range(2 ** d):
        for a in range(d):
            shp[:, c] *= (1.0 + t[:, a]) / 2.0 if (c >> a) & 1 else (1.0 - t[:, a]) / 2.0
    return np.einsum("lc,ecd->eld", shp, space.mesh.corners)


class FESpace:
    def __init__(self, mesh, p, vdim=1, n_q=None):
        if p < 1:
            raise ValueError(f"degree must be >= 1, got {p}")
        if vdim < 1:
            raise ValueError(f"vdim must be >= 1, got {vdim}")
        self.mesh = mesh
        self.p = p
        self.vdim = vdim
        self.dim = mesh.dim
        self.basis = make_basis(p, n_q=n_q)
        (self.element_dofs, self.ndofs_scalar,
         self.num_edges, self.num_faces) = number_dofs(mesh, p)
        self._owner = None
        self._coords = None

    @property
    def ndofs(self):
        return self.vdim * self.ndofs_scalar

    @property
    def nloc(self):
        return (self.p + 1) ** self.dim

    def component(self, x, c):
        ns = self.ndofs_scalar
        return x[c * ns:(c + 1) * ns]

    # first appearance in element-major scan order owns a DoF (fespace.py:247-263)
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
        if self._coords is None:
            coords = element_node_coords(self)
            e, l = self._owners()
            self._coords = coords[e, l]
        return self._coords

    def gather(self, x):
        return x[self.element_dofs]

    def scatter_add(self, xloc):
        return np.bincount(self.element_dofs.ravel(), weights=np.ascontiguousarray(xloc).ravel(),
                           minlength=self.ndofs_scalar)

    def boundary_dof_set(self, attributes=None):
        known = self.mesh.boundary_attributes()
        if attributes is None:
            attributes = known
        else:
            attributes = set(int(a) for a in attributes)
            bad = attributes - known
            if bad:
                raise ValueError(f"unknown boundary attributes {sorted(bad)}")
        bf = self.mesh.boundary_faces
        lat = local_lattice(self.p, self.dim)
        out = []
        for f in range(2 * self.dim):
            axis, side = divmod(f, 2)
            rows = bf[(bf[:, 1] == f) & np.isin(bf[:, 2], list(attributes)), 0]
            if rows.size:
                sel = lat[:, axis] == (self.p if side else 0)
                out.append(self.element_dofs[rows][:, sel].ravel())
        if not out:
            return np.zeros(0, dtype=np.int64)
        return np.unique(np.concatenate(out))

    def expand_dofs(self, scalar_dofs, components=None):
        comps = range(self.vdim) if components is None else components
        ns = self.ndofs_scalar
        return np.concatenate([np.asarray(scalar_dofs) + c * ns for c in comps])

    def project(self, f):
        vals = np.asarray(f(self.node_coords), dtype=np.float64)
        if self.vdim == 1:
            if vals.shape != (self.ndofs_scalar,):
                raise ValueError(f"projection callable returned shape {vals.shape}")
            return vals.copy()
        if vals.shape != (self.ndofs_scalar, self.vdim):
            raise ValueError(f"projection callable returned shape {vals.shape}")
        return vals.T.reshape(-1).copy()
