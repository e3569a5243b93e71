"""The sharded solvers through torch.distributed / NCCL (one process per GPU).
On one GPU (world 1) it checks the cfg3 path's NCCL all-reduce / all-gather
calls; with two or more GPUs also the slab exchanges and the periodic ring.
Not a scaling measurement.
    python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1 tools/nccl_smoke.py"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_03032_b200 import dist_box as D, dist_periodic as DP, geometry, solvers  # noqa: E402


def main():
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group("nccl")
    comm = D.TorchComm()
    cfg = solvers.SolverConfig(rel_tol=1e-8, max_iters=300)
    pr = D.helmholtz_slab_problem(comm, (8, 8, 8), 4, c=10.0)
    x, rep = D.dist_cg(pr["A"], pr["b"], pr["M"], comm, pr["level"].n_own, cfg)
    out = {"world": comm.world, "cfg3_iterations": rep.iterations,
           "cfg3_converged": rep.converged}
    if comm.world >= 2:  # the periodic ring needs two ranks
        m = geometry.cartesian_mesh((4, 4, 8), lows=(-np.pi,) * 3, highs=(np.pi,) * 3,
                                    periodic=(True,) * 3)
        st = DP.DistProjectionStepper(comm, m, 3, k=3, dt=0.02, nu=1.0 / 1600.0)
        st.initialize_from(lambda X: np.stack([np.sin(X[:, 0]) * np.cos(X[:, 1]) * np.cos(X[:, 2]),
                                               -np.cos(X[:, 0]) * np.sin(X[:, 1]) * np.cos(X[:, 2]),
                                               np.zeros(len(X))], axis=1))
        r = st.step()
        out.update(tgv_step=[r.mass_iters, r.pressure_iters, r.helmholtz_iters],
                   energy=st.kinetic_energy())
    if dist.get_rank() == 0:
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
