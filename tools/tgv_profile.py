"""Per-phase timing of device projection steps (cfg5 caller), periodic 3D TGV.

    python tools/tgv_profile.py p n steps
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1910_03032_b200 import geometry, solvers, spaces, timeint  # noqa: E402

p, n, steps = (int(a) for a in sys.argv[1:4])
m = geometry.cartesian_mesh((n, n, n), lows=(-np.pi,) * 3, highs=(np.pi,) * 3, periodic=(True,) * 3)
vs = spaces.FESpace(m, p, vdim=3)
ps = spaces.FESpace(m, p)
geom = geometry.compute_geometric_factors(m, vs.basis.quad)
st = timeint.ProjectionStepper(vs, ps, geom, k=3, dt=0.02, nu=1.0 / 1600.0)


def tgv_u(x):
    X, Y, Z = x[:, 0], x[:, 1], x[:, 2]
    return np.stack([np.sin(X) * np.cos(Y) * np.cos(Z), -np.cos(X) * np.sin(Y) * np.cos(Z),
                     np.zeros_like(X)], axis=1)


st.initialize(vs.project(tgv_u))
for _ in range(3):  # BDF start-up: one Helmholtz LOR hierarchy per order
    st.step()
torch.cuda.synchronize()
# wrap the sub-solves with wall-clock timers
T = {"mass": 0.0, "pressure": 0.0, "helmholtz": 0.0}
orig_cg = timeint.cg


def timed_cg(A, b, precond=None, **kw):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = orig_cg(A, b, precond=precond, **kw)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if A is st.M:
        T["mass"] += dt
    elif A is st.Lp:
        T["pressure"] += dt
    else:
        T["helmholtz"] += dt
    return out


timeint.cg = timed_cg
t0 = time.perf_counter()
for _ in range(steps):
    r = st.step()
torch.cuda.synchronize()
tot = time.perf_counter() - t0
print(f"p={p} n={n} Nv={vs.ndofs} per step {1e3 * tot / steps:.1f} ms; "
      + ", ".join(f"{k} {1e3 * v / steps:.1f} ms" for k, v in T.items()),
      f"its {r.mass_iters}/{r.pressure_iters}/{r.helmholtz_iters}")
# one V-cycle of each preconditioner, device time vs wall time
op, A, pre = st._helmholtz(st.dt and timeint.bdf_coefficients(3).b[0])
for name, P, N in (("pressure", st.pressure_pre, ps.ndofs), ("helmholtz(3 comp)", pre, vs.ndofs)):
    r0 = torch.randn(N, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r0)
    P.apply_into(r0, z)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    for _ in range(20):
        P.apply_into(r0, z)
    e1.record()
    w1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"  {name} V-cycle: device {e0.elapsed_time(e1) / 20:.3f} ms, host enqueue {1e3 * (w1 - w0) / 20:.3f} ms")
