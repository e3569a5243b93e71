"""Scale-mode coarse-solve sweep: CG iterations of the box LOR-PCG against the
number of stationary h-multigrid cycles on the Q1 level (coarse_cycles).

  python tools/coarse_sweep.py small   # golden + cfg3-shape (1M DoFs) cases, RHS in reference numbering
  python tools/coarse_sweep.py full    # cfg3 at 100M DoFs (no reference count exists there)
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1910_03032_b200 import geometry, mfop, solvers, spaces, structured as S  # noqa: E402

CYCLES = [1, 2, 3, 4, 6]


def perm_for(m, p, block=2):
    ref = spaces.FESpace(m, p)
    ids, _ = S.box_lattice_ids(tuple(m.counts), p, block)
    ed = S.lattice_element_dofs(ids, p).numpy()
    perm = np.full(ref.ndofs_scalar, -1, dtype=np.int64)
    perm[ref.element_dofs.ravel()] = ed.ravel()
    return ref, perm


def small():
    cases = [("3d_p4_helmholtz", (4, 4, 4), 0.0, 11, 4, 0, 29, 100),
             ("3d_p7_helmholtz", (4, 4, 4), 0.0, 11, 7, 0, 35, 100),
             ("cfg3s_p4_25", (25, 25, 25), 0.0, 0, 4, 0, 30, 2000),
             ("cfg3s_p7_14", (14, 14, 14), 0.0, 0, 7, 0, 36, 400),
             ("cfg3s_p4_16_pert", (16, 16, 16), 0.05, 1, 4, 0, None, 500),
             ("cfg3s_p7_9_pert", (9, 9, 9), 0.05, 1, 7, 0, None, 100)]
    for name, counts, pert, pseed, p, seed, its_ref, mc in cases:
        m = S.box_mesh(counts, perturb=pert, seed=pseed)
        ref, perm = perm_for(m, p)
        space = S.BoxSpace(m, p, block=2, device=torch.device("cuda"))
        geom = geometry.DeviceGeometry(m, space.basis.quad)
        op = mfop.HelmholtzOperator(space, geom, c=10.0)
        bdr = space.boundary_dof_set()
        A = mfop.ConstrainedOperator(op, bdr)
        b = np.random.default_rng(seed).standard_normal(ref.ndofs)
        b[ref.boundary_dof_set()] = 0.0
        bn = np.empty_like(b)
        bn[perm] = b
        bd = torch.from_numpy(bn).cuda()
        res = {"name": name, "ref": its_ref, "ndofs": ref.ndofs}
        for mcx in (20000, mc):
            pre = S.BoxLORPreconditioner(space, "helmholtz", c=10.0, max_coarse=mcx)
            for k in (CYCLES if mcx == mc else [1]):
                pre.coarse_cycles = k if len(pre.spaces) - 1 > pre.q1_index else 1
                x, rep = solvers.cg(A, bd, precond=pre,
                                    config=solvers.SolverConfig(rel_tol=1e-8, max_iters=300))
                res[f"mc{mcx}_k{k}"] = rep.iterations
            res[f"mc{mcx}_levels"] = [s.ndofs_scalar for s in pre.spaces]
        print(json.dumps(res), flush=True)


def full():
    for p, n in ((4, 116), (7, 66)):
        prob = S.helmholtz_box_problem((n, n, n), p, c=10.0, perturb=0.05, seed=1)
        A, M, b = prob["A"], prob["M"], prob["b"]
        res = {"p": p, "n": n, "levels": M.describe()}
        cfg = solvers.SolverConfig(rel_tol=1e-8, max_iters=300)
        for k in CYCLES:
            M.coarse_cycles = k
            solvers.cg(A, b, precond=M, config=cfg)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            x, rep = solvers.cg(A, b, precond=M, config=cfg)
            torch.cuda.synchronize()
            res[f"k{k}"] = {"its": rep.iterations, "s": round(time.perf_counter() - t0, 3)}
            print(json.dumps(res), flush=True)
        del prob, A, M, b
        torch.cuda.empty_cache()


if __name__ == "__main__":
    {"small": small, "full": full}[sys.argv[1]]()
