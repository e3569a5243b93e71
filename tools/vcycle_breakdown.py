"""Per-kernel breakdown of one scale-mode V-cycle (torch.profiler / CUPTI
kernel records, no ncu): where the cfg3 V-cycle time goes, plus the
preconditioner's per-level byte model.  usage: vcycle_breakdown.py p n [mode lanes]"""
import collections
import json
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_1910_03032_b200 import structured as S  # noqa: E402

p, n = int(sys.argv[1]), int(sys.argv[2])
if len(sys.argv) > 4:  # sweep mode / lanes per block (fb_set_blockilu_pipeline)
    from paper_1910_03032_b200 import _lib
    _lib.check(_lib.lib.fb_set_blockilu_pipeline(int(sys.argv[3]), int(sys.argv[4])))
prob = S.helmholtz_box_problem((n, n, n), p, c=10.0, perturb=0.05, seed=1)
M, b = prob["M"], prob["b"]
out = torch.empty_like(b)
for _ in range(3):
    M.apply_into(b, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    M.apply_into(b, out)
e1.record()
torch.cuda.synchronize()
vms = e0.elapsed_time(e1) / 5
reps = 3
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        M.apply_into(b, out)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        name = ev.name[:90]
        agg[name][0] += 1
        agg[name][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
tot = sum(v[1] for v in agg.values())
print(json.dumps({"p": p, "n": n, "vcycle_ms": round(vms, 3), "kernel_sum_ms": round(tot / reps / 1e3, 3),
                  "levels": M.level_bytes()}, default=int))
for name, (cnt, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{100 * us / tot:5.1f}%  {cnt // reps:4d}/cycle  {us / reps / 1e3:8.3f} ms  {name}")
# launch order of one cycle (durations in us), to attribute launches to levels
seq = [(ev.name[:40], round(ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total, 1))
       for ev in prof.events() if ev.device_type == torch.autograd.DeviceType.CUDA]
print("one cycle:", seq[:len(seq) // reps])
