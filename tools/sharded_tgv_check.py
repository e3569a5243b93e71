"""cfg5 (periodic Taylor-Green, p = 5) through the sharded ring code path on
ONE GPU (in-process ranks): per-step sub-solve counts, velocity and energy
against the single-GPU scale-mode stepper.  Timing is not meaningful.
    python tools/sharded_tgv_check.py p n world steps"""
import gc
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1910_03032_b200 import dist_box as D, dist_periodic as DP, geometry, timeint  # noqa: E402

p, n, world, steps = (int(a) for a in sys.argv[1:5])
m = geometry.cartesian_mesh((n, n, n), lows=(-np.pi,) * 3, highs=(np.pi,) * 3, periodic=(True,) * 3)


def tgv(x):
    X, Y, Z = x[:, 0], x[:, 1], x[:, 2]
    return np.stack([np.sin(X) * np.cos(Y) * np.cos(Z), -np.cos(X) * np.sin(Y) * np.cos(Z),
                     np.zeros_like(X)], axis=1)


one = timeint.BoxProjectionStepper(m, p, k=3, dt=0.02, nu=1.0 / 1600.0)
one.initialize(one.vspace.project(tgv))
ref = []
for _ in range(steps):
    r = one.step()
    ref.append([r.mass_iters, r.pressure_iters, r.helmholtz_iters])
u_ref = one.u.cpu().numpy()
e_ref = one.kinetic_energy()
del one
gc.collect()
torch.cuda.empty_cache()


def fn(comm):
    st = DP.DistProjectionStepper(comm, m, p, k=3, dt=0.02, nu=1.0 / 1600.0)
    st.initialize_from(tgv)
    its = []
    for _ in range(steps):
        r = st.step()
        its.append([r.mass_iters, r.pressure_iters, r.helmholtz_iters])
    parts = st.gather_owned(st.u, 3)
    return its, np.concatenate([q.cpu().numpy() for q in parts]), st.kinetic_energy()


out = D.run_threads(world, fn)
its, u, e = out[0]
print(json.dumps({"p": p, "n": n, "world": world, "single_gpu_iterations": ref,
                  "sharded_iterations": its, "velocity_rel_diff": float(np.linalg.norm(u - u_ref) / np.linalg.norm(u_ref)),
                  "energy": [e_ref, e]}))
