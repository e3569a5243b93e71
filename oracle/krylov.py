"""TEST INFRASTRUCTURE ONLY — numpy/scipy restatement of the reference's
Krylov solvers and LOR V-cycle (solvers.py:108-392), used as the CPU checker
for the device solvers at sizes the golden fixtures do not cover.

  cg          solvers.py:108-169  (preconditioned-residual test, refresh every 50)
  fgmres      solvers.py:172-254  (right preconditioning, MGS, Givens, restarts)
  ilu0        kernels/numba_backend.py:64-103 (IKJ, in place)
  VCycle      solvers.py:321-392  (ILU(0) forward / coarse correction / ILU(0)
              backward; SuperLU bottom)
"""

import numpy as np
import scipy.linalg
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def cg(apply_A, b, precond=None, rel_tol=1e-8, max_iters=500, x0=None, project=None):
    x = np.zeros_like(b) if x0 is None else x0.astype(np.float64, copy=True)
    r = b - apply_A(x)
    if project is not None:
        r = project(r)
    z = precond(r) if precond is not None else r.copy()
    if project is not None:
        z = project(z)
    rz = r @ z
    norm0 = np.sqrt(abs(rz))
    hist = [1.0]
    if norm0 == 0.0:
        return x, 0, hist
    p = z.copy()
    it = 0
    for it in range(1, max_iters + 1):
        Ap = apply_A(p)
        pAp = p @ Ap
        if pAp <= 0.0:
            break
        alpha = rz / pAp
        x += alpha * p
        if it % 50 == 0:
            r = b - apply_A(x)
            if project is not None:
                r = project(r)
        else:
            r -= alpha * Ap
        z = precond(r) if precond is not None else r.copy()
        if project is not None:
            z = project(z)
        rz_new = r @ z
        rel = np.sqrt(abs(rz_new)) / norm0
        hist.append(rel)
        if rel_tol > 0.0 and rel <= rel_tol:
            break
        if rz_new == 0.0:
            break
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, it, hist


def fgmres(apply_A, b, precond=None, rel_tol=1e-8, max_iters=500, restart=50):
    n = b.shape[0]
    x = np.zeros(n)
    r = b - apply_A(x)
    beta0 = np.linalg.norm(r)
    if beta0 == 0.0:
        return x, 0
    target = rel_tol * beta0
    it, done = 0, False
    while it < max_iters and not done:
        beta = np.linalg.norm(r)
        if beta <= target:
            break
        m = restart
        V = np.zeros((m + 1, n))
        Z = np.zeros((m, n))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        j = -1
        for j in range(m):
            if it >= max_iters:
                j -= 1
                break
            it += 1
            Z[j] = precond(V[j]) if precond is not None else V[j]
            w = apply_A(Z[j])
            for i in range(j + 1):
                H[i, j] = V[i] @ w
                w -= H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] > 1e-300:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = (1.0, 0.0) if den == 0.0 else (H[j, j] / den, H[j + 1, j] / den)
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            if abs(g[j + 1]) <= target:
                done = True
                break
        k = j + 1
        if k > 0:
            y = scipy.linalg.solve_triangular(H[:k, :k], g[:k], lower=False)
            x += Z[:k].T @ y
        r = b - apply_A(x)
        if np.linalg.norm(r) <= target:
            done = True
    return x, it


def ilu0(indptr, indices, data):
    """In-place IKJ ILU(0) on sorted CSR; returns -1 or the failing row."""
    n = len(indptr) - 1
    diag = np.empty(n, dtype=np.int64)
    for i in range(n):
        row = indices[indptr[i]:indptr[i + 1]]
        hit = np.flatnonzero(row == i)
        if hit.size == 0:
            return i
        diag[i] = indptr[i] + hit[0]
    pos = {}
    for i in range(n):
        pos = {int(indices[k]): k for k in range(indptr[i], indptr[i + 1])}
        for k in range(indptr[i], indptr[i + 1]):
            c = indices[k]
            if c >= i:
                break
            piv = data[diag[c]]
            if abs(piv) < 1e-300:
                return c
            lik = data[k] / piv
            data[k] = lik
            for kk in range(diag[c] + 1, indptr[c + 1]):
                t = pos.get(int(indices[kk]), -1)
                if t >= 0:
                    data[t] -= lik * data[kk]
        if abs(data[diag[i]]) < 1e-300:
            return i
    return -1


class VCycle:
    """Reference V(1,1) cycle on given level matrices / transfers / orderings."""

    def __init__(self, mats, transfers, orders):
        self.mats = mats
        self.transfers = transfers
        self.smoothers = []
        for A, order in zip(mats[:-1], orders):
            Ap = A[order][:, order].tocsr()
            Ap.sort_indices()
            data = Ap.data.astype(np.float64, copy=True)
            fail = ilu0(Ap.indptr, Ap.indices, data)
            assert fail < 0
            F = sp.csr_matrix((data, Ap.indices, Ap.indptr), shape=A.shape)
            L = (sp.tril(F, k=-1) + sp.eye(A.shape[0])).tocsr()
            U = sp.triu(F).tocsr()
            self.smoothers.append((order, L, U))
        self.bottom = spla.splu(mats[-1].tocsc())

    def _fwd(self, l, r):
        order, L, U = self.smoothers[l]
        out = np.empty_like(r)
        y = spla.spsolve_triangular(L, r[order], lower=True)
        out[order] = spla.spsolve_triangular(U, y, lower=False)
        return out

    def _bwd(self, l, r):
        order, L, U = self.smoothers[l]
        out = np.empty_like(r)
        y = spla.spsolve_triangular(U.T.tocsr(), r[order], lower=True)
        out[order] = spla.spsolve_triangular(L.T.tocsr(), y, lower=False)
        return out

    def cycle(self, l, r):
        if l == len(self.mats) - 1:
            return self.bottom.solve(r)
        A, P = self.mats[l], self.transfers[l]
        x = self._fwd(l, r)
        x = x + P @ self.cycle(l + 1, P.T @ (r - A @ x))
        return x + self._bwd(l, r - A @ x)

    def __call__(self, r):
        return self.cycle(0, r)
