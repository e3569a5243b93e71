"""Scale-mode LOR-PCG on a structured box (cfg3 shapes): setup split,
iterations, time-to-solve.  usage: python tools/box_solve.py p n [max_coarse]"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1910_03032_b200 import solvers, structured as S  # noqa: E402

p, n = int(sys.argv[1]), int(sys.argv[2])
mc = int(sys.argv[3]) if len(sys.argv) > 3 else 20000
t0 = time.perf_counter()
prob = S.helmholtz_box_problem((n, n, n), p, c=10.0, max_coarse=mc)
t1 = time.perf_counter()
cfg = solvers.SolverConfig(rel_tol=1e-8, max_iters=300)
for rep_i in range(2):
    torch.cuda.synchronize()
    ts = time.perf_counter()
    x, rep = solvers.cg(prob["A"], prob["b"], precond=prob["M"], config=cfg)
    torch.cuda.synchronize()
    te = time.perf_counter()
print(json.dumps({"p": p, "n": n, "ndofs": prob["space"].ndofs_scalar, "iterations": rep.iterations,
                  "converged": rep.converged, "solve_s": te - ts, "setup_total_s": t1 - t0,
                  "setup_operator_s": prob["setup_operator_s"],
                  "setup_precond_s": prob["setup_precond_s"], "levels": prob["M"].describe(),
                  "mem_gb": torch.cuda.max_memory_allocated() / 1e9}))
