"""Per-kernel breakdown of cfg3 CG iterations (CUPTI kernel records):
everything outside the operator apply and the V-cycle.  usage: cg_breakdown.py p n"""
import collections
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_1910_03032_b200 import solvers, structured as S  # noqa: E402

p, n = int(sys.argv[1]), int(sys.argv[2])
prob = S.helmholtz_box_problem((n, n, n), p, c=10.0, perturb=0.05, seed=1)
A, M, b = prob["A"], prob["M"], prob["b"]
its = 5
cfg = solvers.SolverConfig(rel_tol=1e-30, max_iters=its)
solvers.cg(A, b, precond=M, config=cfg)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
solvers.cg(A, b, precond=M, config=cfg)
e1.record()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    solvers.cg(A, b, precond=M, config=cfg)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        agg[ev.name[:80]][0] += 1
        agg[ev.name[:80]][1] += ev.device_time_total
tot = sum(v[1] for v in agg.values())
print(f"cg {its} iterations: {e0.elapsed_time(e1):.1f} ms wall (events), kernels {tot / 1e3:.1f} ms")
for name, (cnt, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{100 * us / tot:5.1f}%  {cnt:4d}  {us / 1e3:8.3f} ms  {name}")
