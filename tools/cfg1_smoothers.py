"""cfg1 (2D 16x16 p = 4 Poisson) LOR-PCG with the block and the global ILU(0)
smoothers; TRI_MODE=0|1 picks the triangular-solve mode (sync-free / levels)."""
import sys, time, json, numpy as np, torch
sys.path.insert(0, ".")
from paper_1910_03032_b200 import _lib, geometry, mfop, solvers, spaces
import os
if os.environ.get("TRI_MODE"):
    _lib.check(_lib.lib.fb_set_trisolve_mode(int(os.environ["TRI_MODE"]), int(os.environ.get("TRI_BACKOFF", "0"))))
m = geometry.cartesian_mesh((16, 16))
sp = spaces.FESpace(m, 4)
geom = geometry.DeviceGeometry(m, sp.basis.quad)
op = mfop.setup("stiffness", space=sp, geom=geom, nu=1.0, c=0.0)
bdr = sp.boundary_dof_set()
A = mfop.ConstrainedOperator(op, bdr)
out = {}
for sm in ("block", "global"):
    pre = solvers.LORPreconditioner(sp, "stiffness", dirichlet_attrs="all", smoother=sm)
    b = np.random.default_rng(0).standard_normal(sp.ndofs); b[bdr] = 0.0
    bd = torch.from_numpy(b).cuda()
    cfg = solvers.SolverConfig(rel_tol=1e-8, max_iters=300)
    solvers.cg(A, bd, precond=pre, config=cfg); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        x, rep = solvers.cg(A, bd, precond=pre, config=cfg)
    torch.cuda.synchronize()
    out[sm] = {"its": rep.iterations, "ms": round((time.perf_counter() - t0) / 5 * 1e3, 2)}
print(json.dumps(out))
