"""A/B of the block-ILU sweeps: level-packed TMA ring vs CSR/ELL sweeps on a
structured box (scale mode).  Prints fine-level sweep time, V-cycle time and
the CG iteration count / solve time of each.

    python tools/bilu_ab.py p n
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1910_03032_b200 import _lib, solvers, structured as S  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


p, n = int(sys.argv[1]), int(sys.argv[2])
res = {"p": p, "n": n}
xs = {}
for packed in (0, 1):
    _lib.check(_lib.lib.fb_set_blockilu_packed(packed))
    prob = S.helmholtz_box_problem((n, n, n), p, c=10.0)
    A, M, b = prob["A"], prob["M"], prob["b"]
    sm = M.smoothers[0]
    r = b.clone()
    out = torch.empty_like(b)
    f_ms = timed(lambda: sm.forward_into(r, out))
    b_ms = timed(lambda: sm.backward_into(r, out))
    fw = sm.forward_into(r, torch.empty_like(b)).clone()
    v_ms = timed(lambda: M.apply_into(r, out))
    cfg = solvers.SolverConfig(rel_tol=1e-8, max_iters=300)
    solvers.cg(A, b, precond=M, config=cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, rep = solvers.cg(A, b, precond=M, config=cfg)
    e1.record()
    torch.cuda.synchronize()
    xs[packed] = (fw, x)
    res[f"packed{packed}"] = {"fwd_sweep_ms": round(f_ms, 3), "bwd_sweep_ms": round(b_ms, 3),
                              "vcycle_ms": round(v_ms, 3), "its": rep.iterations,
                              "solve_ms": round(e0.elapsed_time(e1), 1)}
    del prob, A, M, b, sm
    torch.cuda.empty_cache()
res["fwd_bitwise_equal"] = bool(torch.equal(xs[0][0], xs[1][0]))
res["fwd_rel_diff"] = float((xs[0][0] - xs[1][0]).norm() / xs[0][0].norm())
res["x_rel_diff"] = float((xs[0][1] - xs[1][1]).norm() / xs[0][1].norm())
print(json.dumps(res), flush=True)
