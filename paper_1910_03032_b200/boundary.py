"""Boundary surface functionals of the projection method, applied on the device.

The reference evaluates two face integrals per time step of a bounded-domain
``ProjectionStepper`` (timeint.py:310-316, 360):

* ``boundary_normal_flux(space, g)`` (mfop.py:623-684):
  b_i = sum over boundary faces of  int_f psi_i (g . n)
* ``boundary_rotational_rhs(vspace, pspace, u, nu)`` (mfop.py:687-807):
  r_j = -nu * sum over faces of  int_f (n x curl u) . grad psi_j,
  with curl u the one-sided trace of the adjacent element's expansion.

Both are linear: in the face-point values of g, and in u.  Here each is
built ONCE per (space, attributes, n_quad) as a sparse matrix whose per-face
blocks restate the reference formulas (same face quadrature, the same
d-linear corner map, the same outward-normal orientation test), and every
call is one libfbb200 CSR SpMV on the device (``vec.DeviceCSR``):

* normal flux:  N (n_p x nfaces*nqf*d), N[m, (f,q,k)] = psi_m(q) w_q n_k(q);
  the callable g is evaluated on the host at the stacked face points (as the
  reference does face by face), the values go to the device, y = N g.
* rotational rhs:  R (n_p x d*n_v), per face
  R_f = -nu sum_{a,a'} T_a^T diag(K_{a,c,a'}) F_{a'}, where F_{a'} evaluates
  d u_c / d xi_{a'} at the face points, K maps reference gradients to the
  weighted (n x curl u) pulled back through J^{-T}, and T_a evaluates
  d psi / d xi_a.  y = R u.

The per-face sums become CSR rows summed in column order instead of the
reference's face-by-face ``out[...] +=``; results agree to rounding
(tests/test_boundary.py: 1e-12 relative against the reference's functions).
"""

import numpy as np
import scipy.sparse as sp
import torch

from . import device as dev
from . import vec
from .quadrature import build_eval_matrices, gauss_legendre_rule
from .spaces import local_lattice


def _selected_faces(mesh, attributes):
    known = mesh.boundary_attributes()
    attrs = known if attributes is None else set(int(a) for a in attributes)
    bf = np.asarray(mesh.boundary_faces, dtype=np.int64).reshape(-1, 3)
    keep = np.isin(bf[:, 2], sorted(attrs)) if bf.shape[0] else np.zeros(0, dtype=bool)
    return bf[keep]


def _face_points(d, nq1, axis, side):
    """Reference-coordinate face points lambda in [0,1]^d (first in-face axis
    fastest) and the in-face point indices (mfop.py:718-735)."""
    xi, w1 = gauss_legendre_rule(nq1)
    xi, w1 = np.asarray(xi), np.asarray(w1)
    lam = 0.5 * (xi + 1.0)
    in_face = [a for a in range(d) if a != axis]
    if d == 2:
        nqf, wf = nq1, w1
        iq1, iq2 = np.arange(nq1), None
    else:
        nqf = nq1 * nq1
        wf = np.tile(w1, nq1) * np.repeat(w1, nq1)
        iq1, iq2 = np.arange(nqf) % nq1, np.arange(nqf) // nq1
    lams = np.empty((nqf, d))
    lams[:, axis] = float(side)
    lams[:, in_face[0]] = lam[iq1]
    if d == 3:
        lams[:, in_face[1]] = lam[iq2]
    return lams, wf, iq1, iq2, in_face


def _corner_map(corners, lams):
    """Points x and Jacobian d x / d xi (= 0.5 d x / d lambda) of the d-linear
    corner map for a batch of elements: corners (nf, 2^d, d), lams (nqf, d)
    -> x (nf, nqf, d), jac (nf, nqf, d, d) (mfop.py:736-747)."""
    d = lams.shape[1]
    clat = local_lattice(1, d)
    nf, nqf = corners.shape[0], lams.shape[0]
    x = np.zeros((nf, nqf, d))
    dxdl = np.zeros((nf, nqf, d, d))
    for bits, ci in zip(clat, range(clat.shape[0])):
        w = np.where(bits[None, :] == 1, lams, 1.0 - lams)
        corner = corners[:, ci, :]  # (nf, d)
        x += np.prod(w, axis=1)[None, :, None] * corner[:, None, :]
        for a in range(d):
            others = np.prod(np.delete(w, a, axis=1), axis=1)
            sgn = 1.0 if bits[a] else -1.0
            dxdl[:, :, :, a] += sgn * others[None, :, None] * corner[:, None, :]
    return x, 0.5 * dxdl


def _outward(nrm, x, corners):
    """Flip the normals of faces whose mean normal points into the element."""
    centre = corners.mean(axis=1)  # (nf, d)
    s = np.einsum("fk,fk->f", nrm.mean(axis=1), x.mean(axis=1) - centre)
    return np.where((s < 0.0)[:, None, None], -nrm, nrm)


def _face_tensor(mats, d):
    """Rows = face points, columns = element-local lattice index (x fastest):
    prod_b mats[b][q, i_b] (mfop.py:777-781, 791-796)."""
    if d == 2:
        return np.einsum("qi,qj->qji", *mats).reshape(mats[0].shape[0], -1)
    return np.einsum("qi,qj,qk->qkji", *mats).reshape(mats[0].shape[0], -1)


def _face_eval(B, D, BE, DE, axis, side, iq1, iq2, in_face, deriv_axis, d, nqf):
    mats = []
    for b in range(d):
        if b == axis:
            pair = (np.broadcast_to(BE[side], (nqf, BE.shape[1])),
                    np.broadcast_to(DE[side], (nqf, DE.shape[1])))
        elif b == in_face[0]:
            pair = B[iq1], D[iq1]
        else:
            pair = B[iq2], D[iq2]
        mats.append(pair[1] if b == deriv_axis else pair[0])
    return _face_tensor(mats, d)


class NormalFluxMatrix:
    """boundary_normal_flux as a device SpMV (mfop.py:623-684)."""

    def __init__(self, space, attributes=None, n_quad=None):
        mesh = space.mesh
        d, p = space.dim, space.p
        nq = int(n_quad) if n_quad is not None else p + 2
        xi, wq = gauss_legendre_rule(nq)
        B1, _ = build_eval_matrices(space.basis.nodes, np.asarray(xi))
        wq = np.asarray(wq)
        lat = local_lattice(p, d)
        faces = _selected_faces(mesh, attributes)
        self.dim = d
        self.nfaces = faces.shape[0]
        self.ndofs = space.ndofs_scalar
        if d == 2:
            nqf, w2 = nq, wq
            vals = B1
        else:
            nqf = nq * nq
            w2 = np.tile(wq, nq) * np.repeat(wq, nq)
            vals = np.einsum("qi,qj->qij", B1[np.arange(nqf) // nq],
                             B1[np.arange(nqf) % nq]).reshape(nqf, -1)
        self.nqf = nqf
        pts = np.zeros((self.nfaces, nqf, d))
        rows, cols, data = [], [], []
        for f in range(2 * d):
            sel = np.nonzero(faces[:, 1] == f)[0]
            if sel.size == 0:
                continue
            axis, side = divmod(f, 2)
            els = faces[sel, 0]
            lams, _, _, _, in_face = _face_points(d, nq, axis, side)
            cr = mesh.corners[els]
            x, jac = _corner_map(cr, lams)
            if d == 2:
                tan = jac[:, :, :, in_face[0]]
                nrm = np.stack([tan[:, :, 1], -tan[:, :, 0]], axis=2)
            else:
                nrm = np.cross(jac[:, :, :, in_face[0]], jac[:, :, :, in_face[1]])
            nrm = _outward(nrm, x, cr)
            pts[sel] = x
            dofs = space.element_dofs[els][:, lat[:, axis] == (p if side else 0)]  # (nf, nfd)
            # block[m, q, k] = vals[q, m] w[q] n_k(q)
            blk = np.einsum("qm,q,fqk->fmqk", vals, w2, nrm)
            col0 = (sel[:, None] * nqf + np.arange(nqf)[None, :]) * d  # (nf, nqf)
            colidx = col0[:, None, :, None] + np.arange(d)[None, None, None, :]
            rows.append(np.broadcast_to(dofs[:, :, None, None], blk.shape).ravel())
            cols.append(np.broadcast_to(colidx, blk.shape).ravel())
            data.append(blk.ravel())
        self.points = pts.reshape(-1, d)
        ncols = self.nfaces * nqf * d
        if rows:
            A = sp.csr_matrix((np.concatenate(data), (np.concatenate(rows), np.concatenate(cols))),
                              shape=(self.ndofs, ncols))
        else:
            A = sp.csr_matrix((self.ndofs, max(ncols, 1)))
        A.eliminate_zeros()
        self.matrix = A  # host copy (setup product; tests check it against the reference)
        self.nnz = A.nnz
        self._dev = None

    def _device(self):
        if self._dev is None and self.nnz:
            self._dev = vec.DeviceCSR(self.matrix)
        return self._dev

    def apply_values(self, gvals):
        """Device SpMV of face-point values (nfaces*nqf, d) -> (n_p,) device."""
        y = dev.zeros(self.ndofs)
        if self._device() is None:
            return y
        g = dev.to_device(np.ascontiguousarray(gvals, dtype=np.float64).reshape(-1))
        self._device().apply_into(g, y)
        return y

    def __call__(self, g):
        if self.nfaces == 0:
            return dev.zeros(self.ndofs)
        vals = np.asarray(g(self.points), dtype=np.float64)
        if vals.shape != (self.points.shape[0], self.dim):
            raise ValueError(f"flux callable returned shape {vals.shape}, "
                             f"expected ({self.points.shape[0]}, {self.dim})")
        return self.apply_values(vals)


class RotationalMatrix:
    """boundary_rotational_rhs as a device SpMV (mfop.py:687-807)."""

    def __init__(self, vspace, pspace, nu=1.0, attributes=None, n_quad=None):
        mesh = vspace.mesh
        d = vspace.dim
        if vspace.vdim != d or d not in (2, 3):
            raise ValueError("curl needs a 2D or 3D vector velocity space")
        if pspace.mesh is not vspace.mesh or pspace.vdim != 1:
            raise ValueError("pressure space must be scalar on the same mesh")
        nq1 = int(n_quad) if n_quad is not None else max(vspace.p, pspace.p) + 2
        xi, _ = gauss_legendre_rule(nq1)
        xi = np.asarray(xi)
        ends = np.array([-1.0, 1.0])
        Bv, Dv = build_eval_matrices(vspace.basis.nodes, xi)
        Bp, Dp = build_eval_matrices(pspace.basis.nodes, xi)
        BvE, DvE = build_eval_matrices(vspace.basis.nodes, ends)
        BpE, DpE = build_eval_matrices(pspace.basis.nodes, ends)
        faces = _selected_faces(mesh, attributes)
        self.nu = float(nu)
        self.nfaces = faces.shape[0]
        self.np_ = pspace.ndofs
        self.nv = vspace.ndofs_scalar
        rows, cols, data = [], [], []
        for f in range(2 * d):
            sel = np.nonzero(faces[:, 1] == f)[0]
            if sel.size == 0:
                continue
            axis, side = divmod(f, 2)
            els = faces[sel, 0]
            lams, wf, iq1, iq2, in_face = _face_points(d, nq1, axis, side)
            nqf = lams.shape[0]
            cr = mesh.corners[els]
            x, jac = _corner_map(cr, lams)
            jinv = np.linalg.inv(jac)  # (nf, nqf, d, d): [xi_a, x_i]
            if d == 2:
                tan = jac[:, :, :, in_face[0]]
                nrm = np.stack([tan[:, :, 1], -tan[:, :, 0]], axis=2)
            else:
                nrm = np.cross(jac[:, :, :, in_face[0]], jac[:, :, :, in_face[1]])
            nrm = _outward(nrm, x, cr)
            # K[f, q, a, c, a']: coefficient of gref[c, a'] in coeff[a]
            nf = els.shape[0]
            K = np.zeros((nf, nqf, d, d, d))
            for c in range(d):
                for ap in range(d):
                    grads = np.zeros((nf, nqf, d, d))  # [component, x-derivative]
                    grads[:, :, c, :] = jinv[:, :, ap, :]
                    if d == 2:
                        omega = grads[:, :, 1, 0] - grads[:, :, 0, 1]
                        v = omega[:, :, None] * np.stack([nrm[:, :, 1], -nrm[:, :, 0]], axis=2)
                    else:
                        omega = np.stack([grads[:, :, 2, 1] - grads[:, :, 1, 2],
                                          grads[:, :, 0, 2] - grads[:, :, 2, 0],
                                          grads[:, :, 1, 0] - grads[:, :, 0, 1]], axis=2)
                        v = np.cross(nrm, omega)
                    K[:, :, :, c, ap] = np.einsum("fqai,fqi->fqa", jinv, v) * wf[None, :, None]
            Fv = np.stack([_face_eval(Bv, Dv, BvE, DvE, axis, side, iq1, iq2, in_face, a, d, nqf)
                           for a in range(d)])  # (d, nqf, nvloc)
            Tp = np.stack([_face_eval(Bp, Dp, BpE, DpE, axis, side, iq1, iq2, in_face, a, d, nqf)
                           for a in range(d)])  # (d, nqf, nploc)
            # blk[f, m, c, l] = -nu sum_{a, a', q} Tp[a, q, m] K[f, q, a, c, a'] Fv[a', q, l]
            tmp = np.einsum("fqacb,bql->fqacl", K, Fv)
            blk = -self.nu * np.einsum("aqm,fqacl->fmcl", Tp, tmp)
            pd = pspace.element_dofs[els]  # (nf, nploc)
            vd = vspace.element_dofs[els]  # (nf, nvloc)
            colidx = vd[:, None, :] + (np.arange(d) * self.nv)[None, :, None]  # (nf, d, nvloc)
            rows.append(np.broadcast_to(pd[:, :, None, None], blk.shape).ravel())
            cols.append(np.broadcast_to(colidx[:, None, :, :], blk.shape).ravel())
            data.append(blk.ravel())
        if rows:
            A = sp.csr_matrix((np.concatenate(data), (np.concatenate(rows), np.concatenate(cols))),
                              shape=(self.np_, d * self.nv))
        else:
            A = sp.csr_matrix((self.np_, d * self.nv))
        A.eliminate_zeros()
        self.matrix = A  # host copy (setup product; tests check it against the reference)
        self.nnz = A.nnz
        self._dev = None

    def _device(self):
        if self._dev is None and self.nnz:
            self._dev = vec.DeviceCSR(self.matrix)
        return self._dev

    def apply_into(self, u, y, stream=None):
        if self._device() is None:
            y.zero_()
            return y
        return self._device().apply_into(u, y, stream)

    def __call__(self, u):
        ud, host = dev.DeviceIn.get(u)
        y = dev.zeros(self.np_)
        self.apply_into(ud, y)
        return dev.to_host(y) if host else y


# Face matrices are cached ON the space objects they belong to (attribute
# `_fb_face_cache`), so a cached matrix lives exactly as long as its space and
# a new space can never pick up a stale matrix through a recycled id().
_CACHE_ATTR = "_fb_face_cache"


def _cached(owner, key, make):
    cache = getattr(owner, _CACHE_ATTR, None)
    if cache is None:
        cache = {}
        try:
            setattr(owner, _CACHE_ATTR, cache)
        except AttributeError:  # an object without a __dict__: no caching
            return make()
    obj = cache.get(key)
    if obj is None:
        obj = make()
        cache[key] = obj
    return obj


def _attr_key(attributes):
    return None if attributes is None else tuple(sorted(int(a) for a in attributes))


def flux_matrix(space, attributes=None, n_quad=None):
    """The cached NormalFluxMatrix of (space, attributes, n_quad)."""
    key = ("flux", _attr_key(attributes), n_quad)
    return _cached(space, key, lambda: NormalFluxMatrix(space, attributes, n_quad))


def boundary_normal_flux(space, g, attributes=None, n_quad=None):
    """b_i = int over the selected boundary faces of psi_i (g . n)
    (mfop.py:623-684).  Returns a host array, like the reference."""
    return dev.to_host(flux_matrix(space, attributes, n_quad)(g))


def boundary_rotational_rhs(vspace, pspace, u, nu=1.0, attributes=None, n_quad=None):
    """r_j = -nu sum_faces int (n x curl u) . grad psi_j (mfop.py:687-807).
    A device tensor u gives a device result; a host array gives a host array."""
    # keyed on the pressure space too, held strongly by the matrix (M.pspace)
    key = ("rot", id(pspace), float(nu), _attr_key(attributes), n_quad)
    M = _cached(vspace, key, lambda: RotationalMatrix(vspace, pspace, nu, attributes, n_quad))
    if getattr(M, "_pspace_ref", pspace) is not pspace:  # a recycled id(): rebuild
        M = RotationalMatrix(vspace, pspace, nu, attributes, n_quad)
        getattr(vspace, _CACHE_ATTR)[key] = M
    M._pspace_ref = pspace
    return M(u)


def clear_cache(*spaces):
    for sp_ in spaces:
        if hasattr(sp_, _CACHE_ATTR):
            getattr(sp_, _CACHE_ATTR).clear()


__all__ = ["NormalFluxMatrix", "RotationalMatrix", "boundary_normal_flux", "flux_matrix",
           "boundary_rotational_rhs", "clear_cache"]

_ = torch  # device tensors flow through dev/vec
