"""Marginal cost of each pass of the fused kernel: time the kernel with the
arithmetic of one pass skipped (fb_set_fast_skip; results invalid).

    python tools/pass_cost.py [--p 3 4 6 8] [--dofs 1e7]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, nargs="+", default=[3, 4, 6, 8])
    ap.add_argument("--dofs", type=float, default=1e7)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch
    import bench
    from paper_1910_03032_b200 import _lib
    st = torch.cuda.current_stream()

    def t(op, x, y):
        for _ in range(3):
            _lib.check(_lib.lib.fb_operator_apply_part(op.handle, x.data_ptr(), y.data_ptr(), 1,
                                                       st.cuda_stream))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            _lib.check(_lib.lib.fb_operator_apply_part(op.handle, x.data_ptr(), y.data_ptr(), 1,
                                                       st.cuda_stream))
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps

    for p in a.p:
        pr = bench.build_problem(p, target=a.dofs)
        x = torch.randn(pr["N"], dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        base = t(pr["op"], x, y)
        parts = []
        for k in range(1, 13):
            _lib.lib.fb_set_fast_skip(1 << k)
            name = {10: "stores", 11: "S-stores", 12: "line-order-stores"}.get(k, f"P{k}")
            parts.append(f"{name} {base - t(pr['op'], x, y):+.4f}")
        _lib.lib.fb_set_fast_skip(0x3FE)
        allskip = t(pr["op"], x, y)
        _lib.lib.fb_set_fast_skip(0)
        print(f"p={p}: full {base:.4f} ms, all passes skipped {allskip:.4f} ms; saved by skipping: "
              + "  ".join(parts), flush=True)
        del pr


if __name__ == "__main__":
    main()
