"""Time the device ILU(0) sweeps and one LOR V-cycle for a 3D Helmholtz case
under both triangular-solve strategies.

    python tools/bench_trisolve.py --p 4 --n 16
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--n", type=int, default=16)
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_1910_03032_b200 import _lib, geometry, solvers, spaces
    m = geometry.cartesian_mesh((a.n,) * 3)
    sp = spaces.FESpace(m, a.p)
    t0 = time.perf_counter()
    pre = solvers.LORPreconditioner(sp, "helmholtz", c=10.0, dirichlet_attrs="all")
    print(f"N={sp.ndofs} setup {time.perf_counter() - t0:.1f}s levels(L)="
          f"{_lib.lib.fb_trisolve_levels(pre.smoothers[0]._L.handle)}", flush=True)
    r = torch.randn(sp.ndofs, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    sm = pre.smoothers[0]
    for mode, back in ((1, 0), (0, 256)):
        _lib.check(_lib.lib.fb_set_trisolve_mode(mode, back))
        sm.forward_into(r, z)
        pre.apply_into(r, z)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            sm.forward_into(r, z)
        e1.record()
        torch.cuda.synchronize()
        fwd = e0.elapsed_time(e1) / 5
        e0.record()
        for _ in range(3):
            pre.apply_into(r, z)
        e1.record()
        torch.cuda.synchronize()
        vc = e0.elapsed_time(e1) / 3
        print(f"mode={mode} backoff={back}: ILU forward sweep pair {fwd:.3f} ms, V-cycle {vc:.3f} ms",
              flush=True)




def block_mode(p, n):
    import torch
    from paper_1910_03032_b200 import geometry, solvers, spaces
    m = geometry.cartesian_mesh((n,) * 3)
    sp = spaces.FESpace(m, p)
    pre = solvers.LORPreconditioner(sp, "helmholtz", c=10.0, dirichlet_attrs="all", smoother="block")
    r = torch.randn(sp.ndofs, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    sm = pre.smoothers[0]
    for _ in range(2):
        sm.forward_into(r, z)
        pre.apply_into(r, z)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        sm.forward_into(r, z)
    e1.record()
    torch.cuda.synchronize()
    fwd = e0.elapsed_time(e1) / 10
    e0.record()
    for _ in range(10):
        pre.apply_into(r, z)
    e1.record()
    torch.cuda.synchronize()
    print(f"block mode p={p} n={n} N={sp.ndofs}: blocks {sm.nblocks}, forward sweep {fwd:.3f} ms, "
          f"V-cycle {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)


if __name__ == "__main__":
    if "--block" in sys.argv:
        sys.argv.remove("--block")
        a = sys.argv
        block_mode(int(a[a.index("--p") + 1]), int(a[a.index("--n") + 1]))
    else:
        main()
