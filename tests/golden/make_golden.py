"""Generate golden fixtures from the REAL reference (flowbench 0.1.0).

Run in the build container, where /root/reference exists:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py [group ...]

The reference is imported from /root/reference/pkg/src and driven through its
public API (mesh, FESpace, mfop, solvers, lor).  Outputs are small .npz files
in this directory plus manifest.json describing each case; the GPU box never
needs the reference.  Inputs are reproducible from the recorded mesh
parameters and numpy.random.default_rng seeds.
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def ref_modules():
    sys.path.insert(0, REF)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    from flowbench import fespace, lor, mesh, mfop, solvers, stokes  # noqa: F401
    return mesh, fespace, mfop, solvers, lor, stokes


# (name, d, counts, periodic, perturb, p, kind, c, nu, vdim, seed)
APPLY_CASES = []
for _p in (1, 2, 3, 4, 6):
    for _k in ("mass", "stiffness", "helmholtz"):
        APPLY_CASES.append((f"2d_p{_p}_{_k}", 2, (3, 2), None, 0.08, _p, _k, 0.7, 1.3, 1, 5))
for _p in (1, 2, 3, 4):
    for _k in ("mass", "stiffness", "helmholtz"):
        APPLY_CASES.append((f"3d_p{_p}_{_k}", 3, (2, 2, 2), None, 0.08, _p, _k, 0.7, 1.3, 1, 5))
for _p in (5, 6, 7, 8):
    for _k in ("mass", "stiffness", "helmholtz"):
        APPLY_CASES.append((f"3d_p{_p}_{_k}", 3, (3, 2, 2), None, 0.05, _p, _k, 10.0, 1.0, 1, 7))
APPLY_CASES += [
    ("3d_p3_affine_helmholtz", 3, (3, 3, 2), None, 0.0, 3, "helmholtz", 10.0, 1.0, 1, 1),
    ("3d_p2_periodic_helmholtz", 3, (3, 3, 3), (True, True, True), 0.05, 2, "helmholtz", 2.0, 0.5, 1, 2),
    ("3d_p4_periodic_stiffness", 3, (3, 4, 3), (True, False, True), 0.05, 4, "stiffness", 0.0, 1.0, 1, 3),
    ("3d_p3_vector_stiffness", 3, (2, 2, 2), None, 0.08, 3, "stiffness", 0.0, 1.3, 3, 4),
    ("3d_p4_vector_helmholtz", 3, (2, 2, 2), None, 0.08, 4, "helmholtz", 10.0, 1.0, 3, 4),
    ("2d_p3_vector_mass", 2, (3, 2), None, 0.08, 3, "mass", 0.0, 1.0, 2, 0),
    ("cfg1_poisson", 2, (16, 16), None, 0.0, 4, "stiffness", 0.0, 1.0, 1, 0),
    ("2d_p12_helmholtz", 2, (2, 2), None, 0.05, 12, "helmholtz", 1.0, 1.0, 1, 9),
]

# (name, d, counts, periodic, perturb, pv, pp, seed)
MIXED_CASES = [
    ("2d_th3", 2, (3, 2), None, 0.08, 3, 2, 3),
    ("3d_th3", 3, (2, 2, 2), None, 0.08, 3, 2, 3),
    ("3d_th2_periodic", 3, (3, 3, 3), (True,) * 3, 0.05, 2, 1, 4),
    ("3d_th5", 3, (2, 2, 1), None, 0.05, 5, 4, 6),
]


def build(mesh_mod, fes_mod, d, counts, periodic, perturb, p, vdim=1):
    m = mesh_mod.cartesian_mesh(counts, periodic=periodic)
    if perturb:
        m = mesh_mod.perturb_mesh(m, perturb, seed=11)
    sp = fes_mod.FESpace(m, p, vdim=vdim)
    geom = mesh_mod.compute_geometric_factors(m, sp.basis.quad)
    return m, sp, geom


def make_apply():
    mesh, fespace, mfop, _, _, _ = ref_modules()
    out, manifest = {}, []
    for (name, d, counts, periodic, perturb, p, kind, c, nu, vdim, seed) in APPLY_CASES:
        _, sp, geom = build(mesh, fespace, d, counts, periodic, perturb, p, vdim)
        kw = {"mass": {}, "stiffness": {"nu": nu}, "helmholtz": {"c": c, "nu": nu}}[kind]
        op = mfop.setup(kind, space=sp, geom=geom, **kw)
        x = np.random.default_rng(seed).standard_normal(sp.ndofs)
        out[name + "/y"] = op.apply(x)
        # constrained variant (mfop.py:416-433) on the full boundary
        if sp.mesh.boundary_faces.shape[0]:
            bd = sp.expand_dofs(sp.boundary_dof_set())
            out[name + "/yc"] = mfop.ConstrainedOperator(op, bd).apply(x)
        out[name + "/element_dofs_sum"] = np.array([sp.element_dofs.sum(), sp.ndofs_scalar])
        manifest.append(dict(name=name, d=d, counts=counts, periodic=periodic, perturb=perturb,
                             p=p, kind=kind, c=c, nu=nu, vdim=vdim, seed=seed,
                             ndofs=int(sp.ndofs)))
    mixed = []
    for (name, d, counts, periodic, perturb, pv, pp, seed) in MIXED_CASES:
        m, vs, geom = build(mesh, fespace, d, counts, periodic, perturb, pv, vdim=d)
        ps = fespace.FESpace(m, pp)
        G = mfop.GradientOperator(vs, ps, geom)
        D = mfop.DivergenceOperator(vs, ps, geom)
        rng = np.random.default_rng(seed)
        q = rng.standard_normal(ps.ndofs_scalar)
        v = rng.standard_normal(vs.ndofs)
        out[name + "/G"] = G.apply(q)
        out[name + "/Gt"] = G.apply_transpose(v)
        out[name + "/D"] = D.apply(v)
        mixed.append(dict(name=name, d=d, counts=counts, periodic=periodic, perturb=perturb,
                          pv=pv, pp=pp, seed=seed))
    np.savez_compressed(os.path.join(HERE, "apply.npz"), **out)
    return {"apply": manifest, "mixed": mixed}


def make_numbering():
    mesh, fespace, _, _, _, _ = ref_modules()
    cases = [(2, (3, 2), None, 3), (3, (2, 2, 2), None, 3), (3, (3, 2, 4), None, 4),
             (3, (3, 3, 3), (True,) * 3, 3), (2, (3, 4), (True, False), 4),
             (3, (4, 3, 3), (False, True, True), 2), (3, (2, 3, 2), None, 1)]
    out, manifest = {}, []
    for i, (d, counts, periodic, p) in enumerate(cases):
        m = mesh.perturb_mesh(mesh.cartesian_mesh(counts, periodic=periodic), 0.08, seed=11)
        sp = fespace.FESpace(m, p)
        key = f"n{i}"
        out[key + "/element_dofs"] = sp.element_dofs
        out[key + "/boundary"] = sp.boundary_dof_set()
        out[key + "/owner_elem"] = sp.dof_owner_elem
        out[key + "/corners"] = m.corners
        geom = mesh.compute_geometric_factors(m, sp.basis.quad)
        out[key + "/detj"] = geom.detj
        out[key + "/jinv"] = geom.jinv
        manifest.append(dict(key=key, d=d, counts=counts, periodic=periodic, p=p,
                             ndofs=int(sp.ndofs_scalar)))
    np.savez_compressed(os.path.join(HERE, "numbering.npz"), **out)
    return {"numbering": manifest}


# (name, d, counts, perturb, p, kind, c, seeds)
SOLVE_CASES = [
    ("cfg1_poisson", 2, (16, 16), 0.0, 4, "stiffness", 0.0, (0, 1, 2)),
    ("cfg1_helmholtz", 2, (16, 16), 0.0, 4, "helmholtz", 10.0, (0,)),
    ("2d_p7_helmholtz_pert", 2, (6, 5), 0.05, 7, "helmholtz", 10.0, (3,)),
    ("3d_p4_helmholtz", 3, (4, 4, 4), 0.0, 4, "helmholtz", 10.0, (0,)),
    ("3d_p7_helmholtz", 3, (4, 4, 4), 0.0, 7, "helmholtz", 10.0, (0,)),
    ("3d_p2_stiffness_pert", 3, (5, 4, 4), 0.05, 2, "stiffness", 0.0, (1,)),
    ("3d_p3_mass", 3, (3, 3, 3), 0.0, 3, "mass", 0.0, (2,)),
]


def make_solvers():
    mesh, fespace, mfop, solvers, lor, _ = ref_modules()
    out, manifest = {}, []
    for (name, d, counts, perturb, p, kind, c, seeds) in SOLVE_CASES:
        m = mesh.cartesian_mesh(counts)
        if perturb:
            m = mesh.perturb_mesh(m, perturb, seed=11)
        sp_ = fespace.FESpace(m, p)
        geom = mesh.compute_geometric_factors(m, sp_.basis.quad)
        kw = {"mass": {}, "stiffness": {"nu": 1.0}, "helmholtz": {"c": c, "nu": 1.0}}[kind]
        op = mfop.setup(kind, space=sp_, geom=geom, **kw)
        bdr = sp_.boundary_dof_set()
        A = mfop.ConstrainedOperator(op, bdr)
        pre = solvers.LORPreconditioner(sp_, kind, nu=1.0, c=c, dirichlet_attrs="all")
        r = np.random.default_rng(99).standard_normal(sp_.ndofs)
        out[name + "/vcycle_in_seed"] = np.array([99])
        out[name + "/vcycle"] = pre.apply(r)
        sm = pre.smoothers[0]
        out[name + "/ilu_fwd"] = sm.forward(r)
        out[name + "/ilu_bwd"] = sm.backward(r)
        out[name + "/lor_nnz"] = np.array([A_.nnz for _, A_ in pre.levels])
        its = []
        for seed in seeds:
            b = np.random.default_rng(seed).standard_normal(sp_.ndofs)
            b[bdr] = 0.0
            x, rep = solvers.cg(A, b, precond=pre,
                                config=solvers.SolverConfig(rel_tol=1e-8, max_iters=300))
            out[f"{name}/x{seed}"] = x
            out[f"{name}/hist{seed}"] = np.array(rep.residuals)
            its.append(rep.iterations)
        manifest.append(dict(name=name, d=d, counts=counts, perturb=perturb, p=p, kind=kind,
                             c=c, seeds=list(seeds), iterations=its))
    # ILU(0) factor values on the cfg1 finest LOR level (kernels/numba_backend.py:64-103)
    m = mesh.cartesian_mesh((16, 16))
    sp_ = fespace.FESpace(m, 4)
    A = lor.lor_matrix(sp_, "stiffness", constrained=sp_.boundary_dof_set())
    order = solvers._first_touch_ordering(sp_)
    Ap = A[order][:, order].tocsr()
    Ap.sort_indices()
    data = Ap.data.astype(np.float64, copy=True)
    from flowbench.kernels import ilu0_factor
    fail = ilu0_factor(Ap.indptr, Ap.indices, data)
    out["ilu/order"] = order
    out["ilu/indptr"] = Ap.indptr
    out["ilu/indices"] = Ap.indices
    out["ilu/data_in"] = Ap.data
    out["ilu/data_out"] = data
    out["ilu/fail"] = np.array([fail])
    # pure-Neumann Poisson with mean projection (solvers.py:361-362, 384-390)
    m = mesh.perturb_mesh(mesh.cartesian_mesh((8, 8)), 0.05, seed=11)
    sp_ = fespace.FESpace(m, 3)
    geom = mesh.compute_geometric_factors(m, sp_.basis.quad)
    L = mfop.StiffnessOperator(sp_, geom)
    pre = solvers.LORPreconditioner(sp_, "stiffness", pure_neumann=True)
    b = solvers.deflate_mean(np.random.default_rng(5).standard_normal(sp_.ndofs))
    x, rep = solvers.cg(L, b, precond=pre, project=solvers.MeanProjector(),
                        config=solvers.SolverConfig(rel_tol=1e-10, max_iters=300))
    out["neumann/x"] = x
    manifest.append(dict(name="neumann", iterations=[rep.iterations]))
    np.savez_compressed(os.path.join(HERE, "solvers.npz"), **out)
    return {"solvers": manifest}


# cfg3-shape LOR-PCG at ~1M DoFs: (name, counts, perturb, perturb_seed, p, c)
CFG3_CASES = [
    ("cfg3s_p4_25", (25, 25, 25), 0.0, 0, 4, 10.0),
    ("cfg3s_p7_14", (14, 14, 14), 0.0, 0, 7, 10.0),
    ("cfg3s_p4_16_pert", (16, 16, 16), 0.05, 1, 4, 10.0),
    ("cfg3s_p7_9_pert", (9, 9, 9), 0.05, 1, 7, 10.0),
]


def make_cfg3shape():
    """Reference iteration counts (and a solution fingerprint) of the
    Helmholtz LOR-PCG at the cfg3 shape, ~0.3-1M DoFs, b = default_rng(0)
    normal with zero boundary values, rel_tol 1e-8 (app.py:453-496 protocol).
    Perturbed cases use perturb_mesh(m, 0.05, seed=1) like bench.py."""
    import time
    mesh, fespace, mfop, solvers, lor, _ = ref_modules()
    out, manifest = {}, []
    for (name, counts, perturb, pseed, p, c) in CFG3_CASES:
        t0 = time.perf_counter()
        m = mesh.cartesian_mesh(counts)
        if perturb:
            m = mesh.perturb_mesh(m, perturb, seed=pseed)
        sp_ = fespace.FESpace(m, p)
        geom = mesh.compute_geometric_factors(m, sp_.basis.quad)
        op = mfop.HelmholtzOperator(sp_, geom, c=c, nu=1.0)
        bdr = sp_.boundary_dof_set()
        A = mfop.ConstrainedOperator(op, bdr)
        pre = solvers.LORPreconditioner(sp_, "helmholtz", nu=1.0, c=c, dirichlet_attrs="all")
        t1 = time.perf_counter()
        b = np.random.default_rng(0).standard_normal(sp_.ndofs)
        b[bdr] = 0.0
        x, rep = solvers.cg(A, b, precond=pre,
                            config=solvers.SolverConfig(rel_tol=1e-8, max_iters=300))
        t2 = time.perf_counter()
        idx = np.random.default_rng(1).choice(sp_.ndofs, 4096, replace=False)
        out[f"{name}/idx"] = idx
        out[f"{name}/x_sample"] = x[idx]
        out[f"{name}/hist"] = np.array(rep.residuals)
        manifest.append(dict(name=name, counts=list(counts), perturb=perturb, perturb_seed=pseed,
                             p=p, c=c, ndofs=int(sp_.ndofs), iterations=rep.iterations,
                             x_norm=float(np.linalg.norm(x)), setup_s=round(t1 - t0, 1),
                             solve_s=round(t2 - t1, 1)))
        print(manifest[-1], flush=True)
    np.savez_compressed(os.path.join(HERE, "cfg3shape.npz"), **out)
    return {"cfg3shape": manifest}


# periodic boxes (cfg5 shape), LOR-PCG: (name, counts, p, kind, c, pure_neumann, rel_tol)
PERIODIC_CASES = [
    ("per_pn_p5_6", (6, 6, 6), 5, "stiffness", 0.0, True, 1e-10),
    ("per_pn_p3_8", (8, 8, 8), 3, "stiffness", 0.0, True, 1e-10),
    ("per_helm_p4_6", (6, 6, 6), 4, "helmholtz", 10.0, False, 1e-8),
]


def make_periodic():
    """Fully periodic [-pi, pi]^3 boxes (the cfg5 Taylor-Green domain):
    pure-Neumann Poisson with MeanProjector (solvers.py:361-362, 384-390) and
    a Helmholtz solve, reference LORPreconditioner + cg; counts and a solution
    fingerprint for the scale-mode (BoxSpace) periodic path."""
    mesh, fespace, mfop, solvers, lor, _ = ref_modules()
    out, manifest = {}, []
    for (name, counts, p, kind, c, pn, tol) in PERIODIC_CASES:
        m = mesh.cartesian_mesh(counts, lows=(-np.pi,) * 3, highs=(np.pi,) * 3,
                                periodic=(True,) * 3)
        sp_ = fespace.FESpace(m, p, n_q=p + 2)
        geom = mesh.compute_geometric_factors(m, sp_.basis.quad)
        op = mfop.setup(kind, space=sp_, geom=geom, nu=1.0, c=c)
        b = np.random.default_rng(5).standard_normal(sp_.ndofs)
        cfg = solvers.SolverConfig(rel_tol=tol, max_iters=300)
        if pn:
            pre = solvers.LORPreconditioner(sp_, kind, pure_neumann=True)
            b = solvers.deflate_mean(b)
            x, rep = solvers.cg(op, b, precond=pre, project=solvers.MeanProjector(), config=cfg)
        else:
            pre = solvers.LORPreconditioner(sp_, kind, nu=1.0, c=c)
            x, rep = solvers.cg(op, b, precond=pre, config=cfg)
        idx = np.random.default_rng(1).choice(sp_.ndofs, min(4096, sp_.ndofs), replace=False)
        out[f"{name}/idx"] = idx
        out[f"{name}/x_sample"] = x[idx]
        manifest.append(dict(name=name, counts=list(counts), p=p, kind=kind, c=c,
                             pure_neumann=pn, rel_tol=tol, ndofs=int(sp_.ndofs),
                             iterations=rep.iterations))
        print(manifest[-1], flush=True)
    np.savez_compressed(os.path.join(HERE, "periodic.npz"), **out)
    return {"periodic": manifest}


# (name, d, counts, p, alpha_dt)
STOKES_CASES = [
    ("cav2d_p2", 2, (8, 8), 2, None),
    ("cav2d_p4", 2, (8, 8), 4, None),
    ("cav2d_p6", 2, (8, 8), 6, None),
    ("cav3d_p2", 3, (3, 3, 3), 2, None),
    ("cav2d_p3_unsteady", 2, (8, 8), 3, 0.01),
]


def lid(X):
    d = X.shape[1]
    out = np.zeros_like(X)
    out[np.abs(X[:, 1] - 1.0) < 1e-12, 0] = 1.0
    return out


def make_stokes():
    mesh, fespace, mfop, solvers, _, stokes = ref_modules()
    out, manifest = {}, []
    for (name, d, counts, p, adt) in STOKES_CASES:
        m = mesh.cartesian_mesh(counts)
        vs = fespace.FESpace(m, p, vdim=d)
        ps = fespace.FESpace(m, p - 1)
        geom = mesh.compute_geometric_factors(m, vs.basis.quad)
        S = stokes.StokesSystem(vs, ps, geom, nu=1.0, alpha_dt=adt)
        u, pr, rep = S.solve(g=lid, config=solvers.SolverConfig(rel_tol=1e-8, max_iters=200))
        out[name + "/u"] = u
        out[name + "/p"] = pr
        # one application of K and of the block preconditioner
        x = np.random.default_rng(3).standard_normal(S.K.shape[0])
        out[name + "/Kx"] = S.K.apply(x)
        out[name + "/Px"] = S.P.apply(x)
        manifest.append(dict(name=name, d=d, counts=counts, p=p, alpha_dt=adt,
                             iterations=rep.iterations))
    np.savez_compressed(os.path.join(HERE, "stokes.npz"), **out)
    return {"stokes": manifest}


# (name, d, counts, periodic, perturb, p, seed): ConvectionOperator (mfop.py:322-358)
CONV_CASES = [
    ("conv_2d_p3", 2, (4, 3), None, 0.08, 3, 1),
    ("conv_2d_p6", 2, (2, 2), None, 0.05, 6, 2),
    ("conv_3d_p2", 3, (3, 2, 2), None, 0.08, 2, 3),
    ("conv_3d_p4", 3, (2, 2, 2), None, 0.05, 4, 4),
    ("conv_3d_p5_periodic", 3, (3, 3, 3), (True,) * 3, 0.05, 5, 5),
    ("conv_3d_p7", 3, (2, 1, 1), None, 0.05, 7, 6),
]


CURL_CASES = [
    ("curl_2d_p3", 2, (4, 3), None, 0.08, 3, 7),
    ("curl_3d_p2", 3, (3, 2, 2), None, 0.08, 2, 8),
    ("curl_3d_p4_periodic", 3, (3, 3, 3), (True,) * 3, 0.05, 4, 9),
]


def make_extras():
    """Next-row operators of SURVEY 8(f) item 4 (cfg5 projection step)."""
    mesh, fespace, mfop, _, _, _ = ref_modules()
    out, manifest = {}, []
    for (name, d, counts, periodic, perturb, p, seed) in CONV_CASES:
        _, vs, geom = build(mesh, fespace, d, counts, periodic, perturb, p, vdim=d)
        op = mfop.ConvectionOperator(vs, geom)
        u = np.random.default_rng(seed).standard_normal(vs.ndofs)
        out[name + "/y"] = op.apply(u)
        manifest.append(dict(name=name, d=d, counts=counts, periodic=periodic, perturb=perturb,
                             p=p, seed=seed, ndofs=int(vs.ndofs)))
    # cfg5-shaped projection stepping (timeint.py:218-388): periodic 3D
    # Taylor-Green, BDF3/EXT3, equal order (SURVEY 8(c) recorded counts)
    sys.path.insert(0, REF)
    from flowbench import timeint
    tgv = dict(name="tgv3d_p3", counts=(4, 4, 4), p=3, k=3, dt=0.02, nu=1.0 / 1600.0, steps=4)
    m = mesh.cartesian_mesh(tgv["counts"], lows=(-np.pi,) * 3, highs=(np.pi,) * 3,
                            periodic=(True,) * 3)
    vs = fespace.FESpace(m, tgv["p"], vdim=3)
    ps = fespace.FESpace(m, tgv["p"])
    geom = mesh.compute_geometric_factors(m, vs.basis.quad)
    st = timeint.ProjectionStepper(vs, ps, geom, k=tgv["k"], dt=tgv["dt"], nu=tgv["nu"])
    u0 = vs.project(tgv_velocity)
    st.initialize(u0)
    its = []
    for _ in range(tgv["steps"]):
        r = st.step()
        its.append([r.mass_iters, r.pressure_iters, r.helmholtz_iters])
    out["tgv3d_p3/u0"] = u0
    out["tgv3d_p3/u"] = st.u
    out["tgv3d_p3/p"] = st.p
    out["tgv3d_p3/its"] = np.array(its)
    out["tgv3d_p3/energy"] = np.array([st.kinetic_energy()])
    curl = []
    for (name, d, counts, periodic, perturb, p, seed) in CURL_CASES:
        _, vs, geom = build(mesh, fespace, d, counts, periodic, perturb, p, vdim=d)
        op = mfop.CurlCurlOperator(vs, geom, nu=0.7)
        u = np.random.default_rng(seed).standard_normal(vs.ndofs)
        out[name + "/y"] = op.apply(u)
        curl.append(dict(name=name, d=d, counts=counts, periodic=periodic, perturb=perturb,
                         p=p, seed=seed, nu=0.7))
    np.savez_compressed(os.path.join(HERE, "extras.npz"), **out)
    return {"convection": manifest, "curlcurl": curl, "projection": [dict(tgv, counts=list(tgv["counts"]),
                                                        iterations=its)]}


def tgv_velocity(x):
    """3D Taylor-Green initial velocity on [-pi, pi]^3 (vdim = 3 columns)."""
    X, Y, Z = x[:, 0], x[:, 1], x[:, 2]
    return np.stack([np.sin(X) * np.cos(Y) * np.cos(Z), -np.cos(X) * np.sin(Y) * np.cos(Z),
                     np.zeros_like(X)], axis=1)


# (name, d, counts, perturb, p_v, p_p, attributes, n_quad, seed): the boundary
# surface functionals of the bounded-domain projection step (mfop.py:623-807)
BOUNDARY_CASES = [
    ("bnd_2d_p3", 2, (3, 2), 0.08, 3, 3, None, None, 1),
    ("bnd_2d_p4_th", 2, (2, 3), 0.05, 4, 3, (1, 3), None, 2),
    ("bnd_3d_p2", 3, (2, 2, 2), 0.08, 2, 2, None, None, 3),
    ("bnd_3d_p3_nq", 3, (2, 1, 2), 0.05, 3, 3, (2, 5), 6, 4),
]


def flux_field(x):
    """A smooth vector field with nonzero normal flux on every face."""
    d = x.shape[1]
    cols = [np.sin(1.3 * x[:, 0] + 0.2) + x[:, 1] ** 2, np.cos(0.7 * x[:, 1]) - x[:, 0] * x[:, 1]]
    if d == 3:
        cols.append(x[:, 2] * (1.0 + x[:, 0]) + np.sin(x[:, 1]))
        cols[0] = cols[0] + 0.5 * x[:, 2]
    return np.stack(cols, axis=1)


def tgv2d_exact(nu):
    def g(x, t):
        f = np.exp(-2.0 * nu * t)
        X, Y = x[:, 0], x[:, 1]
        return np.stack([np.sin(X) * np.cos(Y) * f, -np.cos(X) * np.sin(Y) * f], axis=1)
    return g


def make_boundary():
    mesh, fespace, mfop, solvers, _, _ = ref_modules()
    from flowbench import timeint
    out, cases = {}, []
    for (name, d, counts, perturb, pv, pp, attrs, nq, seed) in BOUNDARY_CASES:
        m = mesh.perturb_mesh(mesh.cartesian_mesh(counts), perturb, seed=11)
        vs = fespace.FESpace(m, pv, vdim=d)
        ps = fespace.FESpace(m, pp)
        u = np.random.default_rng(seed).standard_normal(vs.ndofs)
        out[name + "/rot"] = mfop.boundary_rotational_rhs(vs, ps, u, nu=0.37, attributes=attrs,
                                                          n_quad=nq)
        out[name + "/flux"] = mfop.boundary_normal_flux(ps, flux_field, attributes=attrs,
                                                        n_quad=nq)
        cases.append(dict(name=name, d=d, counts=counts, perturb=perturb, p_v=pv, p_p=pp,
                          attributes=attrs, n_quad=nq, seed=seed, nu=0.37))
    # bounded-domain projection stepping (timeint.py:218-388): 2D Taylor-Green
    # on [-1, 1]^2 with the exact decaying solution as Dirichlet data (nonzero
    # normal flux and rotational boundary terms), BDF2/EXT2
    proj = dict(name="tgv2d_box_p4", counts=(4, 4), p=4, k=2, dt=0.05, nu=0.05, steps=4,
                perturb=0.05)
    m = mesh.perturb_mesh(mesh.cartesian_mesh(proj["counts"], lows=(-1.0, -1.0),
                                              highs=(1.0, 1.0)), proj["perturb"], seed=11)
    vs = fespace.FESpace(m, proj["p"], vdim=2)
    ps = fespace.FESpace(m, proj["p"])
    geom = mesh.compute_geometric_factors(m, vs.basis.quad)
    g = tgv2d_exact(proj["nu"])
    st = timeint.ProjectionStepper(vs, ps, geom, k=proj["k"], dt=proj["dt"], nu=proj["nu"],
                                   dirichlet=g)
    u0 = vs.project(lambda x: g(x, 0.0))
    st.initialize(u0)
    its = []
    for _ in range(proj["steps"]):
        r = st.step()
        its.append([r.mass_iters, r.pressure_iters, r.helmholtz_iters])
    out["tgv2d_box_p4/u0"] = u0
    out["tgv2d_box_p4/u"] = st.u
    out["tgv2d_box_p4/p"] = st.p
    np.savez_compressed(os.path.join(HERE, "boundary.npz"), **out)
    return {"boundary": cases, "projection_bounded": [dict(proj, counts=list(proj["counts"]),
                                                          iterations=its)]}


GROUPS = {"apply": make_apply, "numbering": make_numbering, "solvers": make_solvers, "stokes": make_stokes,
          "extras": make_extras, "boundary": make_boundary,
          "cfg3shape": make_cfg3shape, "periodic": make_periodic}


def main(argv):
    groups = argv or list(GROUPS)
    path = os.path.join(HERE, "manifest.json")
    manifest = json.load(open(path)) if os.path.exists(path) else {}
    for g in groups:
        manifest.update(GROUPS[g]())
        print("wrote", g)
    with open(path, "w") as f:
        json.dump(manifest, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
