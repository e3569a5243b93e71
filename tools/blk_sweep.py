import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1910_03032_b200 import geometry, mfop, solvers, spaces
for p, n in ((7, 14), (7, 8), (4, 25)):
    m = geometry.cartesian_mesh((n, n, n)); sp = spaces.FESpace(m, p)
    op = mfop.HelmholtzOperator(sp, geometry.DeviceGeometry(m, sp.basis.quad), 10.0)
    bdr = sp.boundary_dof_set(); A = mfop.ConstrainedOperator(op, bdr)
    b = np.random.default_rng(0).standard_normal(sp.ndofs); b[bdr] = 0
    for blk in (1, 2, 3):
        pre = solvers.LORPreconditioner(sp, "helmholtz", c=10.0, dirichlet_attrs="all", block=blk)
        torch.cuda.synchronize(); t = time.time()
        x, rep = solvers.cg(A, b, precond=pre, config=solvers.SolverConfig(rel_tol=1e-8, max_iters=300))
        torch.cuda.synchronize()
        print(f"p={p} n={n} block={blk}: its={rep.iterations} time={time.time()-t:.3f}s", flush=True)
