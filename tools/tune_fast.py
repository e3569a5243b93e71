"""Time every compiled launch shape of the fused Helmholtz kernel per degree.

    python tools/tune_fast.py [--p 2 3 4 ...] [--dofs 1e7]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, nargs="+", default=[2, 3, 4, 5, 6, 7, 8])
    ap.add_argument("--dofs", type=float, default=1e7)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch
    import bench
    from paper_1910_03032_b200 import _lib
    peak, _ = bench.load_peaks()
    for p in a.p:
        pr = bench.build_problem(p, target=a.dofs)
        x = torch.randn(pr["N"], dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        by = bench.algorithmic_bytes(pr["N"], pr["ne"], p)
        res = []
        for v in range(8):
            if _lib.lib.fb_set_fast_config(p, v) != 0:
                continue
            for _ in range(3):
                _lib.check(_lib.lib.fb_operator_apply_part(pr["op"].handle, x.data_ptr(), y.data_ptr(), 1,
                                                           torch.cuda.current_stream().cuda_stream))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                _lib.lib.fb_operator_apply_part(pr["op"].handle, x.data_ptr(), y.data_ptr(), 1,
                                                torch.cuda.current_stream().cuda_stream)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            res.append((v, ms, by / ms / 1e6 / peak))
        _lib.lib.fb_set_fast_config(p, 0)
        print(f"p={p}: " + "  ".join(f"v{v}: {ms:.4f} ms ({fr:.3f})" for v, ms, fr in res), flush=True)
        del pr, x, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
