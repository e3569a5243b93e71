"""cfg3 at full size through the sharded code path on ONE GPU (in-process
ranks, dist_box.ThreadComm): iteration count and solution against the
single-GPU scale-mode solve.  Timing is not meaningful (ranks share the GPU).
    python tools/sharded_cfg3_check.py p n world"""
import gc
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1910_03032_b200 import dist_box as D, solvers, structured as S  # noqa: E402

p, n, world = (int(a) for a in sys.argv[1:4])
counts = (n, n, n)
cfg = solvers.SolverConfig(rel_tol=1e-8, max_iters=300)
mesh = S.box_mesh(counts, perturb=0.05, seed=1)
ref = S.helmholtz_box_problem(counts, p, c=10.0, perturb=0.05, seed=1)  # same mesh as box_mesh
x_ref, rep_ref = solvers.cg(ref["A"], ref["b"], precond=ref["M"], config=cfg)
x_ref = x_ref.cpu().numpy()
N = ref["space"].ndofs_scalar
del ref
gc.collect()
torch.cuda.empty_cache()


def fn(comm):
    pr = D.helmholtz_slab_problem(comm, counts, p, c=10.0, mesh=mesh)
    lv = pr["level"]
    x, rep = D.dist_cg(pr["A"], pr["b"], pr["M"], comm, lv.n_own, cfg)
    return x[:lv.n_own].cpu().numpy(), rep.iterations, pr["M"].q1_sharded


out = D.run_threads(world, fn)
x = np.concatenate([o[0] for o in out])
print(json.dumps({"p": p, "n": n, "dofs": N, "world": world, "single_gpu_iterations": rep_ref.iterations,
                  "sharded_iterations": [o[1] for o in out], "q1_sharded": out[0][2],
                  "solution_rel_diff": float(np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref))}))
