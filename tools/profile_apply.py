"""Small driver for ncu: builds one 3D Helmholtz problem and applies it.

    python tools/profile_apply.py --p 4 --dofs 4e6 --reps 3 [--kind helmholtz]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, nargs="+", default=[4])
    ap.add_argument("--dofs", type=float, default=4e6)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--kind", default="helmholtz")
    a = ap.parse_args()
    import torch
    from paper_1910_03032_b200 import geometry, mfop, spaces
    for p in a.p:
        n = max(2, round((a.dofs ** (1 / 3) - 1) / p))
        m = geometry.perturb_mesh(geometry.cartesian_mesh((n, n, n)), 0.05, seed=1)
        sp = spaces.FESpace(m, p)
        g = geometry.DeviceGeometry(m, sp.basis.quad)
        op = mfop.setup(a.kind, space=sp, geom=g, c=10.0, nu=1.0)
        x = torch.randn(sp.ndofs, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        for _ in range(a.reps):
            op.apply_into(x, y)
        torch.cuda.synchronize()
        print(f"p={p} N={sp.ndofs} ne={m.num_elements} ok", flush=True)


if __name__ == "__main__":
    main()
