"""TEST INFRASTRUCTURE ONLY — CPU baseline runner for bench.py.

The reference's Helmholtz apply (mfop.py:237-244: gather, values + grads,
qpt scaling, values_t + grads_t, bincount scatter) restated with the
reference's own numpy-backend contraction style (kernels/numpy_backend.py:6-18,
matmul per axis) and run over element chunks on a thread pool, so the CPU
baseline can use every host core.  It is timed beside the GPU path and is
never part of the product.
"""

import concurrent.futures as cf

import numpy as np

from . import sumfact


def _contract3(x, m0, m1, m2):
    ne, n2, n1, n0 = x.shape
    t = np.matmul(x.reshape(-1, n0), m0.T).reshape(ne, n2, n1, m0.shape[0])
    t = np.matmul(m1, t)  # (ne, n2, q1, q0)
    t = np.matmul(m2, t.reshape(ne, n2, -1)).reshape(ne, m2.shape[0], m1.shape[0], m0.shape[0])
    return t


class HelmholtzCPU:
    """y = (c M + L) x on the CPU; `threads` workers over element chunks."""

    def __init__(self, space, geom, c, nu, threads=1):
        self.ed = space.element_dofs
        self.ns = space.ndofs_scalar
        self.n = space.p + 1
        self.B, self.D = space.basis.eval_matrices_at(geom.rule.points)
        self.q = self.B.shape[0]
        self.wdet = c * sumfact.mass_factor(geom.detj, geom.w)
        self.stiff = sumfact.stiffness_factor(geom.detj, geom.jinv, geom.w, nu)
        self.threads = max(1, int(threads))
        ne = self.ed.shape[0]
        nch = self.threads * 4 if self.threads > 1 else 1
        bounds = np.linspace(0, ne, nch + 1).astype(int)
        self.chunks = [(a, b) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
        self.pool = cf.ThreadPoolExecutor(self.threads) if self.threads > 1 else None
        try:
            from threadpoolctl import threadpool_limits
            self._limit = threadpool_limits(limits=1 if self.threads > 1 else None)
        except Exception:
            self._limit = None

    def _chunk(self, x, a, b):
        n, q = self.n, self.q
        B, D = self.B, self.D
        loc = x[self.ed[a:b]].reshape(b - a, n, n, n)
        u = _contract3(loc, B, B, B).reshape(b - a, -1)
        g = [_contract3(loc, D, B, B).reshape(b - a, -1),
             _contract3(loc, B, D, B).reshape(b - a, -1),
             _contract3(loc, B, B, D).reshape(b - a, -1)]
        f = sumfact.sym_apply(self.stiff[a:b], g)
        fu = (u * self.wdet[a:b]).reshape(b - a, q, q, q)
        Bt, Dt = B.T, D.T
        out = _contract3(fu, Bt, Bt, Bt)
        out = out + _contract3(f[0].reshape(b - a, q, q, q), Dt, Bt, Bt)
        out = out + _contract3(f[1].reshape(b - a, q, q, q), Bt, Dt, Bt)
        out = out + _contract3(f[2].reshape(b - a, q, q, q), Bt, Bt, Dt)
        return out.reshape(b - a, -1)

    def __call__(self, x):
        if self.pool is None:
            parts = [self._chunk(x, a, b) for a, b in self.chunks]
        else:
            parts = list(self.pool.map(lambda ab: self._chunk(x, *ab), self.chunks))
        return sumfact.scatter_add(self.ed, np.concatenate(parts, axis=0), self.ns)

    def close(self):
        if self.pool is not None:
            self.pool.shutdown()
