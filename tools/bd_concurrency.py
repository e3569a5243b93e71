import sys, time, json, numpy as np, torch
sys.path.insert(0, ".")
from paper_1910_03032_b200 import geometry, solvers, structured as S
n, p = int(sys.argv[1]), 5
m = geometry.cartesian_mesh((n, n, n), lows=(-np.pi,)*3, highs=(np.pi,)*3, periodic=(True,)*3)
sp = S.BoxSpace(m, p, block=2, device=torch.device("cuda"))
cyc = S.BoxLORPreconditioner(sp, "helmholtz", nu=1/1600, c=50.0)
P = solvers.BlockDiagonalPreconditioner(cyc, 3, sp.ndofs)
r = torch.randn(3 * sp.ndofs, dtype=torch.float64, device="cuda"); out = torch.empty_like(r)
def t(reps=5):
    P.apply_into(r, out); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): P.apply_into(r, out)
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / reps
res = {"n": n, "concurrent_ms": t()}
par, P._par = P._par, None
res["sequential_ms"] = t()
res["single_cycle_ms"] = res["sequential_ms"] / 3
print(json.dumps(res))
