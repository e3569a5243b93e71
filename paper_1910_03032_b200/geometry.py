"""Tensor-product meshes and Q1 geometric factors (host-side setup).

Array-level restatement of the reference mesh contract (mesh.py:17-267):
elements are numbered x-fastest, corners are lexicographic with bit a set on
the high side of axis a, periodic directions identify vertex classes modulo
the cell count, boundary faces carry attribute 2*axis+side+1.  Unlike the
reference generator (a Python loop over elements) everything here is
vectorised, so the 10^7-element meshes of the benchmark build in seconds.
For the operator kernels at scale the factors are computed on the device
(``fb_operator_create_geom``); ``compute_geometric_factors`` is the host
path used for small meshes and for drop-in parity with the reference.
"""

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Mesh:
    dim: int
    vertices: np.ndarray
    elements: np.ndarray
    corners: np.ndarray
    boundary_faces: np.ndarray
    periodic: tuple = ()
    counts: tuple = ()  # structured cell counts (generator meshes)

    @property
    def num_vertices(self):
        return self.vertices.shape[0]

    @property
    def num_elements(self):
        return self.elements.shape[0]

    def boundary_attributes(self):
        if self.boundary_faces.shape[0] == 0:
            return set()
        return set(int(a) for a in np.unique(self.boundary_faces[:, 2]))


def local_face_corners(dim, face):
    axis, side = divmod(face, 2)
    return [c for c in range(2 ** dim) if ((c >> axis) & 1) == side]


def cartesian_mesh(counts, lows=None, highs=None, periodic=None):
    counts = tuple(int(c) for c in counts)
    d = len(counts)
    if d not in (2, 3):
        raise ValueError(f"dimension must be 2 or 3, got {d}")
    if any(c < 1 for c in counts):
        raise ValueError(f"cell counts must be positive, got {counts}")
    lows = tuple(float(v) for v in (lows if lows is not None else (0.0,) * d))
    highs = tuple(float(v) for v in (highs if highs is not None else (1.0,) * d))
    periodic = tuple(bool(b) for b in (periodic if periodic is not None else (False,) * d))
    if any(h <= lo for lo, h in zip(lows, highs)):
        raise ValueError("highs must exceed lows")
    if any(periodic[a] and counts[a] < 3 for a in range(d)):
        raise ValueError("periodic directions need at least 3 cells")

    nva = [counts[a] if periodic[a] else counts[a] + 1 for a in range(d)]
    grid1d = [np.linspace(lows[a], highs[a], counts[a] + 1) for a in range(d)]
    strides = np.cumprod([1] + nva[:-1])

    # vertex classes, x fastest
    idx = np.indices(nva[::-1]).reshape(d, -1)[::-1]  # idx[a] = coordinate along axis a
    vertices = np.stack([grid1d[a][idx[a]] for a in range(d)], axis=1)

    # cells, x fastest
    cells = np.indices(counts[::-1]).reshape(d, -1)[::-1]  # (d, ne)
    ne = cells.shape[1]
    nc = 2 ** d
    elements = np.zeros((ne, nc), dtype=np.int64)
    corners = np.zeros((ne, nc, d))
    for c in range(nc):
        vid = np.zeros(ne, dtype=np.int64)
        for a in range(d):
            ia = cells[a] + ((c >> a) & 1)
            corners[:, c, a] = grid1d[a][ia]
            if periodic[a]:
                ia = ia % counts[a]
            vid += ia * strides[a]
        elements[:, c] = vid

    e_ids, f_ids, attrs = [], [], []
    for a in range(d):
        if periodic[a]:
            continue
        for side in (0, 1):
            sel = np.flatnonzero(cells[a] == (counts[a] - 1 if side else 0))
            e_ids.append(sel)
            f_ids.append(np.full(sel.size, 2 * a + side))
            attrs.append(np.full(sel.size, 2 * a + side + 1))
    if e_ids:
        bf = np.stack([np.concatenate(e_ids), np.concatenate(f_ids), np.concatenate(attrs)], axis=1)
        bf = bf[np.lexsort((bf[:, 2], bf[:, 1], bf[:, 0]))].astype(np.int64)
    else:
        bf = np.zeros((0, 3), dtype=np.int64)
    return Mesh(d, vertices, elements, corners, bf, periodic, counts)


def perturb_mesh(mesh, amplitude, seed=0):
    """Random vertex displacement scaled by the smallest cell extent; the
    boundary of non-periodic directions stays put (mesh.py:149-171)."""
    rng = np.random.default_rng(seed)
    d = mesh.dim
    disp = rng.uniform(-amplitude, amplitude, size=mesh.vertices.shape)
    extent = mesh.corners.max(axis=1) - mesh.corners.min(axis=1)
    disp *= extent.min()
    if mesh.boundary_faces.shape[0]:
        fixed = np.zeros(mesh.num_vertices, dtype=bool)
        bf = mesh.boundary_faces
        for f in range(2 * d):
            sel = bf[bf[:, 1] == f, 0]
            if sel.size:
                fixed[mesh.elements[sel][:, local_face_corners(d, f)].ravel()] = True
        disp[fixed] = 0.0
    return Mesh(d, mesh.vertices + disp, mesh.elements, mesh.corners + disp[mesh.elements],
                mesh.boundary_faces.copy(), mesh.periodic, mesh.counts)


@dataclass
class GeometricFactors:
    rule: object
    xq: np.ndarray
    jac: np.ndarray
    detj: np.ndarray
    jinv: np.ndarray
    w: np.ndarray = field(repr=False)


def tensor_points(pts, d):
    """(nq^d, d) reference coordinates, x fastest."""
    g = np.indices((len(pts),) * d).reshape(d, -1)[::-1]
    return np.stack([pts[g[a]] for a in range(d)], axis=1)


def tensor_weights(w1, d):
    if d == 2:
        return np.einsum("j,i->ji", w1, w1).ravel()
    return np.einsum("k,j,i->kji", w1, w1, w1).ravel()


def q1_shape(ref, d):
    """Multilinear shape values (nq, 2^d) and gradients (nq, 2^d, d)."""
    nq = ref.shape[0]
    N = np.ones((nq, 2 ** d))
    dN = np.ones((nq, 2 ** d, d))
    for c in range(2 ** d):
        for a in range(d):
            hi = (c >> a) & 1
            val = (1.0 + ref[:, a]) / 2.0 if hi else (1.0 - ref[:, a]) / 2.0
            der = 0.5 if hi else -0.5
            N[:, c] *= val
            for b in range(d):
                dN[:, c, b] *= der if a == b else val
    return N, dN


def _inverse_and_det(jac, d):
    a = jac
    if d == 2:
        det = a[..., 0, 0] * a[..., 1, 1] - a[..., 0, 1] * a[..., 1, 0]
        inv = np.empty_like(a)
        inv[..., 0, 0] = a[..., 1, 1]
        inv[..., 0, 1] = -a[..., 0, 1]
        inv[..., 1, 0] = -a[..., 1, 0]
        inv[..., 1, 1] = a[..., 0, 0]
    else:
        det = (a[..., 0, 0] * (a[..., 1, 1] * a[..., 2, 2] - a[..., 1, 2] * a[..., 2, 1])
               - a[..., 0, 1] * (a[..., 1, 0] * a[..., 2, 2] - a[..., 1, 2] * a[..., 2, 0])
               + a[..., 0, 2] * (a[..., 1, 0] * a[..., 2, 1] - a[..., 1, 1] * a[..., 2, 0]))
        inv = np.empty_like(a)
        for i in range(3):
            for j in range(3):
                r0, r1 = [k for k in range(3) if k != j]
                c0, c1 = [k for k in range(3) if k != i]
                # adjugate entry (i, j) = cofactor (j, i)
                inv[..., i, j] = ((-1) ** (i + j)) * (a[..., r0, c0] * a[..., r1, c1]
                                                      - a[..., r0, c1] * a[..., r1, c0])
    inv /= det[..., None, None]
    return det, inv


def compute_geometric_factors(mesh, rule):
    d = mesh.dim
    ref = tensor_points(rule.points, d)
    N, dN = q1_shape(ref, d)
    xq = np.einsum("qc,ecd->eqd", N, mesh.corners)
    jac = np.einsum("qcb,ecd->eqdb", dN, mesh.corners)
    detj, jinv = _inverse_and_det(jac, d)
    if np.any(detj <= 0.0):
        raise ValueError("element mapping is not orientation preserving (det J <= 0)")
    return GeometricFactors(rule, xq, jac, detj, jinv, tensor_weights(rule.weights, d))


class DeviceGeometry:
    """Geometric factors evaluated on the device, never stored on the host.

    Stands in for ``GeometricFactors`` when building operators on large
    meshes: the operator uploads ``mesh.corners`` once and the factor kernel
    (``fb_operator_create_geom``) evaluates the Q1 map, determinant, inverse
    and the operator factors per quadrature point directly into device
    memory.  The host arrays of ``GeometricFactors`` are produced lazily only
    if something asks for them.
    """

    def __init__(self, mesh, rule):
        self.mesh = mesh
        self.rule = rule
        self._host = None

    @property
    def num_elements(self):
        return self.mesh.num_elements

    def _materialise(self):
        if self._host is None:
            self._host = compute_geometric_factors(self.mesh, self.rule)
        return self._host

    @property
    def xq(self):
        return self._materialise().xq

    @property
    def jac(self):
        return self._materialise().jac

    @property
    def detj(self):
        return self._materialise().detj

    @property
    def jinv(self):
        return self._materialise().jinv

    @property
    def w(self):
        return tensor_weights(self.rule.weights, self.mesh.dim)
