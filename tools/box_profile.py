"""Per-phase timing of the scale-mode LOR-PCG pieces on a structured box.
usage: python tools/box_profile.py p n"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1910_03032_b200 import device as dev, geometry, mfop, structured as S  # noqa: E402

p, n = int(sys.argv[1]), int(sys.argv[2])
if len(sys.argv) > 3:
    from paper_1910_03032_b200 import _lib
    _lib.lib.fb_set_blockilu_pipeline(int(sys.argv[3]), int(sys.argv[4]) if len(sys.argv) > 4 else 0)
T = {}
t = time.perf_counter()
mesh = S.box_mesh((n, n, n), perturb=0.05, seed=1)
T["mesh"] = time.perf_counter() - t; t = time.perf_counter()
space = S.BoxSpace(mesh, p, block=2, device=dev.device())
torch.cuda.synchronize()
T["space"] = time.perf_counter() - t; t = time.perf_counter()
ed = space.element_dofs
T["element_dofs_host"] = time.perf_counter() - t; t = time.perf_counter()
r = mfop.restriction(space)
T["restriction"] = time.perf_counter() - t; t = time.perf_counter()
geom = geometry.DeviceGeometry(mesh, space.basis.quad)
op = mfop.HelmholtzOperator(space, geom, c=10.0)
torch.cuda.synchronize()
T["operator"] = time.perf_counter() - t; t = time.perf_counter()
bdr = space.boundary_dof_set()
A = mfop.ConstrainedOperator(op, bdr)
T["boundary"] = time.perf_counter() - t; t = time.perf_counter()
M = S.BoxLORPreconditioner(space, "helmholtz", c=10.0)
T["precond"] = time.perf_counter() - t


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


N = space.ndofs_scalar
x = torch.randn(N, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
P = {"apply_constrained": timeit(lambda: A.apply_into(x, y)), "vcycle": timeit(lambda: M.apply_into(x, y))}
for lev in range(len(M.levels)):
    Al = M._A[lev]
    nl = M.spaces[lev].ndofs_scalar
    a = torch.randn(nl, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    c = torch.empty_like(a)
    P[f"L{lev}_residual"] = timeit(lambda: Al.residual_into(a, a, b))
    if lev < len(M.levels) - 1:
        sm = M.smoothers[lev]
        P[f"L{lev}_smooth_fwd"] = timeit(lambda: sm.forward_into(a, b))
        P[f"L{lev}_smooth_bwd"] = timeit(lambda: sm.backward_into(a, b))
        nc = M.spaces[lev + 1].ndofs_scalar
        cc = torch.randn(nc, dtype=torch.float64, device="cuda")
        P[f"L{lev}_prolong"] = timeit(lambda: M._P[lev].apply_into(cc, b))
        P[f"L{lev}_restrict"] = timeit(lambda: M._Pt[lev].apply_into(a, cc))
print(json.dumps({"p": p, "n": n, "N": N, "setup_s": T, "ms": P}, indent=1))
