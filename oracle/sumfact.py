"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference operator apply.

Follows, per component:
  gather           fespace.py:282-284   x[element_dofs]
  1D contractions  kernels/numpy_backend.py:6-18 (matmul / einsum per axis),
                   the numba backend (numba_backend.py:7-61) computes the same
  values/grads     mfop.py:56-95
  qpt factors      mfop.py:129-166
  scatter_add      fespace.py:286-292   np.bincount (ascending flat order)
  operators        mfop.py:190-319
  constrained      mfop.py:428-433
Inputs are plain arrays, so the oracle works with spaces built by either the
reference or the product package.
"""

import numpy as np

SYM = {2: [(0, 0), (0, 1), (1, 1)], 3: [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]}


def tensor(x, mats):
    """out[e, c, b, a] = sum m2[c,k] m1[b,j] m0[a,i] x[e,k,j,i] (d = len(mats));
    mats = (m0, m1[, m2]) act on axes (last, middle[, first]) — the
    apply_tensor_{2d,3d} contract (kernels/__init__.py:57-68)."""
    if len(mats) == 2:
        m0, m1 = mats
        return np.einsum("bj,eji->ebi", m1, np.einsum("ai,eji->eja", m0, x))
    m0, m1, m2 = mats
    t = np.einsum("ai,ekji->ekja", m0, x)
    t = np.einsum("bj,ekja->ekba", m1, t)
    return np.einsum("ck,ekba->ecba", m2, t)


class Eval:
    """values / grads / values_t / grads_t (mfop.py:34-95)."""

    def __init__(self, B, D, d):
        self.B, self.D, self.d = np.asarray(B), np.asarray(D), d
        self.n = self.B.shape[1]
        self.q = self.B.shape[0]

    def _loc(self, v):
        return v.reshape((v.shape[0],) + (self.n,) * self.d)

    def _qp(self, v):
        return v.reshape((v.shape[0],) + (self.q,) * self.d)

    def values(self, loc):
        return tensor(self._loc(loc), [self.B] * self.d).reshape(loc.shape[0], -1)

    def grads(self, loc):
        x = self._loc(loc)
        out = []
        for m in range(self.d):
            mats = [self.D if a == m else self.B for a in range(self.d)]
            out.append(tensor(x, mats).reshape(loc.shape[0], -1))
        return out

    def values_t(self, f):
        return tensor(self._qp(f), [self.B.T] * self.d).reshape(f.shape[0], -1)

    def grads_t(self, fs):
        out = 0.0
        for m in range(self.d):
            mats = [self.D.T if a == m else self.B.T for a in range(self.d)]
            out = out + tensor(self._qp(fs[m]), mats)
        return out.reshape(fs[0].shape[0], -1)


def gather(element_dofs, x):
    return x[element_dofs]


def scatter_add(element_dofs, xloc, ndofs):
    return np.bincount(element_dofs.ravel(), weights=np.ascontiguousarray(xloc).ravel(),
                       minlength=ndofs)


def mass_factor(detj, w):
    return detj * w[None, :]


def stiffness_factor(detj, jinv, w, nu):
    d = jinv.shape[-1]
    wdet = mass_factor(detj, w)
    out = np.empty(wdet.shape + (len(SYM[d]),))
    for k, (a, b) in enumerate(SYM[d]):
        s = np.zeros_like(wdet)
        for m in range(d):
            s += jinv[..., a, m] * jinv[..., b, m]
        out[..., k] = nu * wdet * s
    return out


def grad_factor(detj, jinv, w):
    wdet = mass_factor(detj, w)
    d = jinv.shape[-1]
    out = np.empty(wdet.shape + (d, d))
    for c in range(d):
        for m in range(d):
            out[..., c, m] = wdet * jinv[..., m, c]
    return out


def sym_apply(stiff, gs):
    d = len(gs)
    W = {}
    for k, (a, b) in enumerate(SYM[d]):
        W[a, b] = W[b, a] = stiff[..., k]
    out = []
    for a in range(d):
        acc = W[a, 0] * gs[0]
        for b in range(1, d):
            acc = acc + W[a, b] * gs[b]
        out.append(acc)
    return out


def square_apply(kind, element_dofs, ndofs_scalar, vdim, B, D, d, x, wdet=None, stiff=None):
    """Mass / stiffness / Helmholtz on a vdim-component SoA vector."""
    ev = Eval(B, D, d)
    ns = ndofs_scalar
    y = np.empty_like(x)
    for c in range(vdim):
        loc = gather(element_dofs, x[c * ns:(c + 1) * ns])
        out = 0.0
        if kind in ("mass", "helmholtz"):
            out = ev.values_t(ev.values(loc) * wdet)
        if kind in ("stiffness", "helmholtz"):
            out = out + ev.grads_t(sym_apply(stiff, ev.grads(loc)))
        y[c * ns:(c + 1) * ns] = scatter_add(element_dofs, out, ns)
    return y


def gradient_apply(v_dofs, nsv, p_dofs, nsp, Bv, Dv, Bp, Dp, d, grad, q):
    evp = Eval(Bp, Dp, d)
    evv = Eval(Bv, Dv, d)
    gs = evp.grads(gather(p_dofs, q))
    out = np.empty(d * nsv)
    for c in range(d):
        f = sum(grad[..., c, m] * gs[m] for m in range(d))
        out[c * nsv:(c + 1) * nsv] = scatter_add(v_dofs, evv.values_t(f), nsv)
    return out


def gradient_transpose_apply(v_dofs, nsv, p_dofs, nsp, Bv, Dv, Bp, Dp, d, grad, v):
    evp = Eval(Bp, Dp, d)
    evv = Eval(Bv, Dv, d)
    fs = None
    for c in range(d):
        vals = evv.values(gather(v_dofs, v[c * nsv:(c + 1) * nsv]))
        terms = [grad[..., c, m] * vals for m in range(d)]
        fs = terms if fs is None else [a + b for a, b in zip(fs, terms)]
    return scatter_add(p_dofs, evp.grads_t(fs), nsp)


def divergence_apply(v_dofs, nsv, p_dofs, nsp, Bv, Dv, Bp, Dp, d, grad, u):
    evp = Eval(Bp, Dp, d)
    evv = Eval(Bv, Dv, d)
    f = None
    for c in range(d):
        gs = evv.grads(gather(v_dofs, u[c * nsv:(c + 1) * nsv]))
        term = sum(grad[..., c, m] * gs[m] for m in range(d))
        f = term if f is None else f + term
    return scatter_add(p_dofs, evp.values_t(f), nsp)


def convection_apply(element_dofs, ns, B, D, d, jinv, wdet, u):
    """N(u)_i = int ((u . grad) u) . phi_i  (mfop.py:322-358): values and
    physical gradients of every component at the qpts, then values_t."""
    ev = Eval(B, D, d)
    vals, gphys = [], {}
    for c in range(d):
        loc = gather(element_dofs, u[c * ns:(c + 1) * ns])
        vals.append(ev.values(loc))
        gs = ev.grads(loc)
        for k in range(d):
            gphys[c, k] = sum(jinv[..., m, k] * gs[m] for m in range(d))
    out = np.empty(d * ns)
    for c in range(d):
        conv = sum(vals[k] * gphys[c, k] for k in range(d))
        out[c * ns:(c + 1) * ns] = scatter_add(element_dofs, ev.values_t(conv * wdet), ns)
    return out


def curlcurl_apply(element_dofs, ns, B, D, d, jinv, wdet, nu, u):
    """int nu (curl u) . (curl v) (mfop.py:381-413)."""
    ev = Eval(B, D, d)
    wd = nu * wdet
    gphys = {}
    for c in range(d):
        gs = ev.grads(gather(element_dofs, u[c * ns:(c + 1) * ns]))
        for k in range(d):
            gphys[c, k] = sum(jinv[..., m, k] * gs[m] for m in range(d))
    out = np.empty(d * ns)
    if d == 2:
        om = wd * (gphys[1, 0] - gphys[0, 1])
        for c, (k, sign) in enumerate([(1, -1.0), (0, 1.0)]):
            fs = [sign * jinv[..., m, k] * om for m in range(d)]
            out[c * ns:(c + 1) * ns] = scatter_add(element_dofs, ev.grads_t(fs), ns)
        return out
    om = [wd * (gphys[2, 1] - gphys[1, 2]), wd * (gphys[0, 2] - gphys[2, 0]),
          wd * (gphys[1, 0] - gphys[0, 1])]
    eps = np.zeros((3, 3, 3))
    for a, b, c in [(0, 1, 2), (1, 2, 0), (2, 0, 1)]:
        eps[a, b, c] = 1.0
        eps[a, c, b] = -1.0
    for c in range(d):
        t = [None] * d
        for b in range(d):
            terms = [eps[a, b, c] * om[a] for a in range(d) if eps[a, b, c] != 0.0]
            t[b] = sum(terms) if terms else None
        fs = [sum(jinv[..., m, b] * t[b] for b in range(d) if t[b] is not None) for m in range(d)]
        out[c * ns:(c + 1) * ns] = scatter_add(element_dofs, ev.grads_t(fs), ns)
    return out


def make_curlcurl(vspace, geom, nu=1.0):
    B, D = eval_matrices(vspace, geom.rule.points)
    wdet = mass_factor(geom.detj, geom.w)
    return lambda u: curlcurl_apply(vspace.element_dofs, vspace.ndofs_scalar, B, D, vspace.dim,
                                    geom.jinv, wdet, nu, u)


def make_convection(vspace, geom):
    B, D = eval_matrices(vspace, geom.rule.points)
    wdet = mass_factor(geom.detj, geom.w)
    return lambda u: convection_apply(vspace.element_dofs, vspace.ndofs_scalar, B, D, vspace.dim,
                                      geom.jinv, wdet, u)


def constrained_apply(apply, constrained, x):
    xi = x.copy()
    xi[constrained] = 0.0
    y = apply(xi)
    y[constrained] = x[constrained]
    return y


# -- convenience: operators from space-like objects ---------------------------

def eval_matrices(space, points):
    return space.basis.eval_matrices_at(points)


def make_square(kind, space, geom, c=0.0, nu=1.0):
    """Closure x -> y of the reference operator on (space, geom)."""
    B, D = eval_matrices(space, geom.rule.points)
    wdet = stiff = None
    if kind in ("mass", "helmholtz"):
        wdet = mass_factor(geom.detj, geom.w)
        if kind == "helmholtz":
            wdet = c * wdet
    if kind in ("stiffness", "helmholtz"):
        stiff = stiffness_factor(geom.detj, geom.jinv, geom.w, nu)
    ed = space.element_dofs
    return lambda x: square_apply(kind, ed, space.ndofs_scalar, space.vdim, B, D, space.dim, x,
                                  wdet, stiff)


def make_mixed(kind, vspace, pspace, geom):
    Bv, Dv = eval_matrices(vspace, geom.rule.points)
    Bp, Dp = eval_matrices(pspace, geom.rule.points)
    G = grad_factor(geom.detj, geom.jinv, geom.w)
    args = (vspace.element_dofs, vspace.ndofs_scalar, pspace.element_dofs, pspace.ndofs_scalar,
            Bv, Dv, Bp, Dp, vspace.dim, G)
    fn = {"gradient": gradient_apply, "divergence": divergence_apply,
          "gradient_t": gradient_transpose_apply}[kind]
    return lambda x: fn(*args, x)
