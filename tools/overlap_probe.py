"""Element kernel: full vs arithmetic only vs memory only (all passes skipped).
The arithmetic-only leg needs the diagnostic build: `git apply
tools/micro/nomem.patch` (skip bit 15 drops the factor / x / y traffic; it
changes code generation, so never keep it in the product build), rebuild,
run, `git apply -R`.  Without the patch the arith_only column equals full."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1910_03032_b200 import _lib  # noqa: E402

st = torch.cuda.current_stream()
degs = [int(a) for a in sys.argv[1:]] or [2, 3, 4, 5, 6, 7, 8]


def t(h, x, y, reps=20):
    for _ in range(3):
        _lib.check(_lib.lib.fb_operator_apply_part(h, x.data_ptr(), y.data_ptr(), 1, st.cuda_stream))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        _lib.check(_lib.lib.fb_operator_apply_part(h, x.data_ptr(), y.data_ptr(), 1, st.cuda_stream))
    b.record(st)
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / reps, 4)


for p in degs:
    pr = bench.build_problem(p)
    x = torch.randn(pr["N"], dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    out = {"p": p}
    for name, mask in (("full", 0), ("arith_only", 1 << 15), ("memory_only", 0x3FE)):
        _lib.lib.fb_set_fast_skip(mask)
        out[name] = t(pr["op"].handle, x, y)
    _lib.lib.fb_set_fast_skip(0)
    print(json.dumps(out), flush=True)
    del pr, x, y
    torch.cuda.empty_cache()
