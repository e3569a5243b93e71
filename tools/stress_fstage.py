"""Stress the staged-factor launch variants on small meshes (single thread)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1910_03032_b200 import _lib, geometry, mfop, structured as S

variants = {2: [0, 3], 3: [0, 5], 4: [0, 6, 3], 5: [0, 5], 6: [0, 4]}
for p, vs in variants.items():
    for counts in [(1, 1, 1), (2, 1, 1), (3, 4, 4), (3, 4, 8), (5, 3, 7), (9, 9, 9)]:
        m = S.box_mesh(counts, perturb=0.05, seed=1)
        sp = S.BoxSpace(m, p, device=torch.device("cuda"))
        op = mfop.HelmholtzOperator(sp, geometry.DeviceGeometry(m, sp.basis.quad), c=10.0)
        x = torch.randn(sp.ndofs, dtype=torch.float64, device="cuda")
        ref = None
        for v in vs:
            _lib.lib.fb_set_fast_config(p, v)
            for _ in range(20):
                y = torch.empty_like(x)
                op.apply_into(x, y)
            torch.cuda.synchronize()
            if ref is None:
                ref = y.clone()
            d = float((y - ref).abs().max())
            if d > 1e-12 * float(ref.abs().max()):
                print("MISMATCH", p, counts, v, d, flush=True)
        print("ok", p, counts, flush=True)
