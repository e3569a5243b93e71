import sys, os
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1910_03032_b200 import dist_box as D, solvers, structured as S, _lib
mode = int(sys.argv[1]) if len(sys.argv) > 1 else -1
if mode >= 0:
    _lib.lib.fb_set_fast_config(4, mode)
if os.environ.get("BILU_MODE"):
    _lib.lib.fb_set_blockilu_pipeline(int(os.environ["BILU_MODE"]), 0)
counts, p, world = (3, 4, 8), 4, int(os.environ.get("WORLD", "2"))
mesh = S.box_mesh(counts, perturb=0.05, seed=1)
cfg = solvers.SolverConfig(rel_tol=1e-8, max_iters=300)
if os.environ.get("WITH_REF"):
    ref = S.helmholtz_box_problem(counts, p, c=10.0, max_coarse=100)
    x_ref, rep_ref = solvers.cg(ref["A"], ref["b"], precond=ref["M"], config=cfg)
    print("ref", rep_ref.iterations, flush=True)
def fn(comm):
    pr = D.helmholtz_slab_problem(comm, counts, p, c=10.0, max_coarse=100, mesh=mesh)
    lv = pr["level"]
    y = torch.empty_like(pr["b"])
    pr["A"].apply_into(pr["b"], y)
    torch.cuda.synchronize()
    print(comm.rank, "apply ok", flush=True)
    x, rep = D.dist_cg(pr["A"], pr["b"], pr["M"], comm, lv.n_own, cfg)
    return rep.iterations
print(D.run_threads(world, fn))
