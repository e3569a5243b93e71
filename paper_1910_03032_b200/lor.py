"""Low-order-refined (LOR) companions of high-order spaces (host setup).

Contract of the reference's ``lor`` module (lor.py:32-131): the nodal lattice
of a degree-p space is a mesh of p^d Q1 sub-cells per element whose vertices
ARE the space's DoFs, so the Q1 matrix assembled on it (2-point Gauss per
direction) is indexed by the parent numbering; constrained rows/columns are
zeroed in-pattern with a unit diagonal; nodal interpolation between degrees
keeps explicit zeros.  The matrices are built once on the host with numpy /
scipy.sparse and moved to the device by the solvers (``sparse.DeviceCSR``).
"""

import numpy as np
import scipy.sparse as sp

from .geometry import compute_geometric_factors
from .quadrature import GAUSS_LEGENDRE, build_eval_matrices, quadrature_rule
from .spaces import element_node_coords

_SYM = {2: [(0, 0), (0, 1), (1, 1)], 3: [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]}


def sub_cell_local_ids(p, d):
    """(p^d, 2^d) local lattice ids of the nodal sub-cells, corners lexicographic."""
    n = p + 1
    cells = np.indices((p,) * d).reshape(d, -1)[::-1]  # cells[a] = index along axis a
    base = sum(cells[a] * n ** a for a in range(d))
    offs = [sum(((c >> a) & 1) * n ** a for a in range(d)) for c in range(2 ** d)]
    return (base[:, None] + np.asarray(offs)[None, :]).astype(np.int64)


def sub_cell_connectivity(space):
    sub = sub_cell_local_ids(space.p, space.dim)
    return space.element_dofs[:, sub].reshape(-1, 2 ** space.dim)


class _SubCellMesh:
    """Just enough of a mesh for compute_geometric_factors."""

    def __init__(self, dim, corners):
        self.dim = dim
        self.corners = corners


def _q1_local_matrices(kind, corners, nu, c):
    """Per-sub-cell Q1 matrices with the 2-point Gauss rule (as mfop.assemble
    does for a Q1 space, mfop.py:496-528)."""
    d = corners.shape[-1]
    rule = quadrature_rule(GAUSS_LEGENDRE, 2)
    geom = compute_geometric_factors(_SubCellMesh(d, corners), rule)
    B, D = build_eval_matrices(np.array([-1.0, 1.0]), rule.points)
    if d == 2:
        Bf = np.kron(B, B)
        Gf = np.stack([np.kron(B, D), np.kron(D, B)], axis=2)
    else:
        Bf = np.kron(B, np.kron(B, B))
        Gf = np.stack([np.kron(B, np.kron(B, D)), np.kron(B, np.kron(D, B)),
                       np.kron(D, np.kron(B, B))], axis=2)
    wdet = geom.detj * geom.w[None, :]
    loc = None
    if kind in ("mass", "helmholtz"):
        wm = wdet if kind == "mass" else c * wdet
        loc = np.einsum("qi,eq,qj->eij", Bf, wm, Bf, optimize=True)
    if kind in ("stiffness", "helmholtz"):
        ne, nq = wdet.shape
        W = np.empty((ne, nq, d, d))
        for a, b in _SYM[d]:
            s = np.zeros_like(wdet)
            for m in range(d):
                s += geom.jinv[..., a, m] * geom.jinv[..., b, m]
            W[..., a, b] = W[..., b, a] = nu * wdet * s
        st = np.einsum("qia,eqab,qjb->eij", Gf, W, Gf, optimize=True)
        loc = st if loc is None else loc + st
    return loc


def lor_matrix(space, kind, nu=1.0, c=0.0, constrained=None):
    """Q1 mass/stiffness/helmholtz matrix on the nodal sub-cell mesh,
    assembled in C++ (fb_lor_assemble_host) directly into CSR."""
    if kind not in ("mass", "stiffness", "helmholtz"):
        raise ValueError(f"unsupported LOR kind {kind!r}")
    if space.vdim != 1:
        raise ValueError("LOR meshes are built from scalar spaces")
    import ctypes as C
    from . import _lib
    ed = np.ascontiguousarray(space.element_dofs, dtype=np.int64)
    corners = np.ascontiguousarray(space.mesh.corners, dtype=np.float64)
    nodes = np.ascontiguousarray(space.basis.nodes, dtype=np.float64)
    cons = np.ascontiguousarray(np.zeros(0) if constrained is None else constrained,
                                dtype=np.int64)
    ns = space.ndofs_scalar
    pi, px, pd = C.c_void_p(), C.c_void_p(), C.c_void_p()
    nnz = _lib.lib.fb_lor_assemble_host(space.dim, space.p, ed.shape[0], ns, _lib.ptr(ed),
                                        _lib.ptr(corners), _lib.ptr(nodes), _lib.KIND[kind],
                                        float(nu), float(c), cons.size, _lib.ptr(cons),
                                        C.byref(pi), C.byref(px), C.byref(pd))
    if nnz < 0:
        _lib.check(int(-nnz))
    try:
        indptr = np.ctypeslib.as_array(C.cast(pi, C.POINTER(C.c_int64)), shape=(ns + 1,)).copy()
        indices = np.ctypeslib.as_array(C.cast(px, C.POINTER(C.c_int64)), shape=(max(nnz, 1),))[:nnz].copy()
        data = np.ctypeslib.as_array(C.cast(pd, C.POINTER(C.c_double)), shape=(max(nnz, 1),))[:nnz].copy()
    finally:
        for ptr_ in (pi, px, pd):
            _lib.lib.fb_host_free(ptr_)
    return sp.csr_matrix((data, indices, indptr), shape=(ns, ns))


def lor_matrix_numpy(space, kind, nu=1.0, c=0.0, constrained=None):
    """numpy assembly of the same matrix (reference-shaped; kept as a
    cross-check of the C++ assembler, tests/test_solvers_cpu.py)."""
    if kind not in ("mass", "stiffness", "helmholtz"):
        raise ValueError(f"unsupported LOR kind {kind!r}")
    if space.vdim != 1:
        raise ValueError("LOR meshes are built from scalar spaces")
    d, p = space.dim, space.p
    sub = sub_cell_local_ids(p, d)
    conn = space.element_dofs[:, sub].reshape(-1, 2 ** d)
    corners = element_node_coords(space)[:, sub, :].reshape(-1, 2 ** d, d)
    loc = _q1_local_matrices(kind, corners, float(nu), float(c))
    nl = 2 ** d
    rows = np.repeat(conn, nl, axis=1).ravel()
    cols = np.tile(conn, (1, nl)).ravel()
    ns = space.ndofs_scalar
    A = sp.coo_matrix((loc.ravel(), (rows, cols)), shape=(ns, ns)).tocsr()
    A.sort_indices()
    if constrained is not None and len(constrained):
        A = constrain_matrix(A, constrained)
    return A


def constrain_matrix(A, dofs):
    """Zero constrained rows and columns, unit diagonal, pattern kept."""
    dofs = np.asarray(dofs, dtype=np.int64)
    A = A.tocsr(copy=True)
    A.sort_indices()
    mask = np.zeros(A.shape[0], dtype=bool)
    mask[dofs] = True
    row_of = np.repeat(np.arange(A.shape[0]), np.diff(A.indptr))
    kill = mask[row_of] | mask[A.indices]
    A.data[kill] = 0.0
    diag_hit = kill & (row_of == A.indices)
    A.data[diag_hit] = 1.0
    missing = dofs[~np.isin(dofs, row_of[diag_hit])]
    if missing.size:  # constrained rows without a stored diagonal
        A = (A + sp.csr_matrix((np.ones(missing.size), (missing, missing)), shape=A.shape)).tocsr()
        A.sort_indices()
    return A


def nodal_interpolation(fine, coarse):
    """Coarse nodal basis at each fine DoF's lattice position in its owner
    element; explicit zeros are kept (lor.py:102-123)."""
    if fine.mesh is not coarse.mesh and fine.mesh.num_elements != coarse.mesh.num_elements:
        raise ValueError("spaces must share the parent mesh")
    B1, _ = build_eval_matrices(coarse.basis.nodes, fine.basis.nodes)
    Bloc = B1
    for _ in range(fine.dim - 1):
        Bloc = np.kron(Bloc, B1)
    ns = fine.ndofs_scalar
    nc = coarse.nloc
    rows = np.repeat(np.arange(ns), nc)
    cols = coarse.element_dofs[fine.dof_owner_elem].ravel()
    vals = Bloc[fine.dof_owner_local].ravel()
    P = sp.coo_matrix((vals, (rows, cols)), shape=(ns, coarse.ndofs_scalar)).tocsr()
    P.sum_duplicates()
    return P


def coarse_q1_interpolation(space):
    from .spaces import FESpace
    return nodal_interpolation(space, FESpace(space.mesh, 1))


def degree_ladder(p):
    degs = [p]
    while degs[-1] > 1:
        degs.append(max(1, (degs[-1] + 1) // 2))
    return degs


def first_touch_ordering(space):
    """DoFs in order of first appearance in the element-major scan
    (solvers.py:257-266)."""
    flat = space.element_dofs.ravel()
    _, first = np.unique(flat, return_index=True)
    return flat[np.sort(first)]
