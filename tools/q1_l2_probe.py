"""p = 1 element kernel after different L2 states (CUDA events): back to back,
after the E->L sum, after a 512 MB write, after a 512 MB read."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1910_03032_b200 import _lib  # noqa: E402

st = torch.cuda.current_stream()
junk = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
pr = bench.build_problem(1)
x = torch.randn(pr["N"], dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
h = pr["op"].handle


def part(k):
    _lib.check(_lib.lib.fb_operator_apply_part(h, x.data_ptr(), y.data_ptr(), k, st.cuda_stream))


def timed(before, reps=10):
    ts = []
    for _ in range(reps):
        before()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        part(1)
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return round(ts[len(ts) // 2], 4)


for _ in range(3):
    part(0)
out = {"after_kernel": timed(lambda: part(1)), "after_scatter": timed(lambda: part(2)),
       "after_write": timed(lambda: junk.fill_(1)), "after_read": timed(lambda: junk.sum()),
       "after_nothing": timed(lambda: None)}
print(json.dumps(out))
