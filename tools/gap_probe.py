"""Where does the full apply's time beyond the element kernel go?  Per degree:
element kernel alone (back to back), E->L sum alone, full apply back to back,
and full apply after an L2 thrash (the sweep's situation).  CUDA events."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1910_03032_b200 import _lib  # noqa: E402

degs = [int(a) for a in sys.argv[1:]] or [2, 3, 4, 5, 6, 7, 8]
st = torch.cuda.current_stream()
junk = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10, thrash=False):
    ts = []
    for _ in range(reps):
        if thrash:
            junk.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return round(ts[len(ts) // 2], 4)


for p in degs:
    pr = bench.build_problem(p)
    x = torch.randn(pr["N"], dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    h = pr["op"].handle

    def part(k):
        return lambda: _lib.check(_lib.lib.fb_operator_apply_part(h, x.data_ptr(), y.data_ptr(),
                                                                  k, st.cuda_stream))
    for _ in range(3):
        part(0)()
    out = {"p": p, "N": pr["N"], "kernel": timed(part(1)), "scatter": timed(part(2)),
           "full": timed(part(0)), "kernel_thrash": timed(part(1), thrash=True),
           "full_thrash": timed(part(0), thrash=True)}
    g, nb, ne = (torch.zeros(1, dtype=torch.int32) for _ in range(3))
    _lib.lib.fb_last_fast_launch(g.data_ptr(), nb.data_ptr(), ne.data_ptr())
    out.update(grid=int(g), nbatch=int(nb), ne_batch=int(ne))
    print(json.dumps(out), flush=True)
    del pr, x, y
    torch.cuda.empty_cache()
