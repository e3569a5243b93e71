"""TEST INFRASTRUCTURE ONLY — times the REAL reference (oracle/_ref) on the host.

Used by bench.py for the reference arm (`--impl reference`) and for the GPU
line's `cpu_baseline` / LOR-PCG comparisons.  Runs the unmodified flowbench
0.1.0 installed by oracle/build_ref.py, through its public API and stock code
path:

* apply: `cartesian_mesh` + `perturb_mesh(0.05, seed=1)`, `FESpace(m, p,
  n_q=p+2)`, `compute_geometric_factors`, `HelmholtzOperator(space, geom,
  c=10, nu=1).apply(x)` (mfop.py:225-244 -> kernels/numba_backend.py:30-61),
  timed like app.py:532-540 `_time_call` (one warm call, then repeats);
* lor_pcg: `cg(ConstrainedOperator(H, bdr), b, LORPreconditioner(space,
  "helmholtz", c, dirichlet_attrs="all"), SolverConfig(rel_tol=1e-8,
  max_iters=300))` exactly as app.py:453-496 drives it (setup and solve timed
  separately).

The backend is `FLOWBENCH_BACKEND=numba` (the reference default; its kernels
are serial `@njit`) and the process is pinned to one thread for
numba / OpenMP / OpenBLAS, except for the `--impl reference` arm, which allows
all host threads (`--threads`); the reference's kernels are serial, so `cores`
= 1 either way.  This module never imports the
product package; run it as a subprocess:

    python -m oracle.ref_bench apply --target 120000 --steps 3 --warmup 1
    python -m oracle.ref_bench pcg --cases cfg1,p4_16,p7_8
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

REF_ENV = {"FLOWBENCH_BACKEND": "numba", "NUMBA_NUM_THREADS": "1", "OMP_NUM_THREADS": "1",
           "OPENBLAS_NUM_THREADS": "1", "MKL_NUM_THREADS": "1",
           "NUMBA_CACHE_DIR": "/tmp/fb_ref_numba_cache"}

# LOR-PCG cases: name -> (counts, p, kind, c, perturb)
PCG_CASES = {
    "cfg1": ((16, 16), 4, "stiffness", 0.0, 0.0),
    "p4_16": ((16, 16, 16), 4, "helmholtz", 10.0, 0.0),
    "p7_8": ((8, 8, 8), 7, "helmholtz", 10.0, 0.0),
    "p4_25": ((25, 25, 25), 4, "helmholtz", 10.0, 0.0),
    "p7_14": ((14, 14, 14), 7, "helmholtz", 10.0, 0.0),
}


def _import_reference():
    for k, v in REF_ENV.items():
        os.environ.setdefault(k, v)
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref", "site"))
    import flowbench  # noqa: F401
    from flowbench import fespace, mesh, mfop, solvers
    assert os.path.abspath(flowbench.__file__).startswith(os.path.join(ROOT, "oracle", "_ref")), \
        flowbench.__file__
    return mesh, fespace, mfop, solvers


def mesh_cells(p, target):
    return max(2, round((target ** (1.0 / 3.0) - 1.0) / p))


def apply_problems(target, degrees, c=10.0, nu=1.0):
    import numpy as np
    mesh, fespace, mfop, _ = _import_reference()
    probs = []
    for p in degrees:
        n = mesh_cells(p, target)
        m = mesh.perturb_mesh(mesh.cartesian_mesh((n, n, n)), 0.05, seed=1)
        sp = fespace.FESpace(m, p, n_q=p + 2)
        geom = mesh.compute_geometric_factors(m, sp.basis.quad)
        op = mfop.HelmholtzOperator(sp, geom, c, nu=nu)
        x = np.random.default_rng(0).standard_normal(sp.ndofs)
        op.apply(x)  # warm caches and the numba JIT (app.py:533)
        probs.append({"p": p, "n": n, "op": op, "x": x, "dofs": int(sp.ndofs)})
    return probs


def apply_sweep(target=120_000, degrees=range(1, 9), steps=3, warmup=1, threads=1):
    """One step = one reference Helmholtz apply per degree.  Returns the
    sweep GDoF/s (total DoFs / total seconds) and per-degree figures."""
    t0 = time.perf_counter()
    probs = apply_problems(target, list(degrees))
    setup = time.perf_counter() - t0
    for _ in range(warmup):
        for pr in probs:
            pr["op"].apply(pr["x"])
    per = {pr["p"]: 0.0 for pr in probs}
    for _ in range(steps):
        for pr in probs:
            ts = time.perf_counter()
            pr["op"].apply(pr["x"])
            per[pr["p"]] += time.perf_counter() - ts
    tot_dofs = steps * sum(pr["dofs"] for pr in probs)
    tot_s = sum(per.values())
    return {
        "value": tot_dofs / tot_s / 1e9, "unit": "GDoF/s", "seconds": tot_s, "steps": steps,
        "warmup": warmup, "setup_s": round(setup, 2), "cores": 1, "threads_allowed": threads,
        "kind": "reference",
        "per_p": {str(pr["p"]): {"dofs": pr["dofs"], "cells": pr["n"],
                                 "ms_per_apply": round(1e3 * per[pr["p"]] / steps, 3),
                                 "mdofs": round(pr["dofs"] * steps / per[pr["p"]] / 1e6, 4)}
                  for pr in probs},
        "sample": (f"reference flowbench 0.1.0 (oracle/_ref) HelmholtzOperator(c=10, nu=1).apply, "
                   f"p=1..8, ~{target / 1e3:.0f}k DoFs per degree (n^3 perturbed cube), "
                   f"FLOWBENCH_BACKEND=numba, {threads} host thread(s) allowed to numba / OpenMP / "
                   f"BLAS; the reference's @njit kernels are serial, so it uses one core "
                   f"(cores = 1); {steps} timed sweep(s) after {warmup} warm-up"),
    }


def lor_pcg(names=("cfg1", "p4_16", "p7_8")):
    import numpy as np
    mesh, fespace, mfop, solvers = _import_reference()
    out = {}
    for name in names:
        counts, p, kind, c, perturb = PCG_CASES[name]
        t0 = time.perf_counter()
        m = mesh.cartesian_mesh(counts)
        if perturb:
            m = mesh.perturb_mesh(m, perturb, seed=1)
        sp = fespace.FESpace(m, p, n_q=p + 2)
        geom = mesh.compute_geometric_factors(m, sp.basis.quad)
        op = mfop.setup(kind, space=sp, geom=geom, nu=1.0, c=c)
        bdr = sp.boundary_dof_set()
        A = mfop.ConstrainedOperator(op, bdr)
        pre = solvers.LORPreconditioner(sp, kind, nu=1.0, c=c, dirichlet_attrs="all")
        setup_s = time.perf_counter() - t0
        b = np.random.default_rng(0).standard_normal(sp.ndofs)
        b[bdr] = 0.0
        cfg = solvers.SolverConfig(rel_tol=1e-8, max_iters=300)
        A.apply(b)  # numba JIT of the contraction kernels outside the timed solve
        pre.apply(b)
        t1 = time.perf_counter()
        x, rep = solvers.cg(A, b, precond=pre, config=cfg)
        t2 = time.perf_counter()
        out[name] = {"dofs": int(sp.ndofs), "counts": list(counts), "p": p, "kind": kind, "c": c,
                     "iterations": rep.iterations, "converged": bool(rep.converged),
                     "setup_s": round(setup_s, 3), "solve_s": round(t2 - t1, 4),
                     "x_norm": float(np.linalg.norm(x))}
    return out


def thread_env(threads):
    env = dict(REF_ENV)
    for k in ("NUMBA_NUM_THREADS", "OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        env[k] = str(threads)
    return env


def run_subprocess(args, timeout=1800, threads=1):
    """Run this module in a fresh interpreter with `threads` host threads
    allowed (1: single-threaded); parsed JSON."""
    import subprocess
    env = dict(os.environ)
    env.update(thread_env(threads))
    args = list(args) + ["--threads", str(threads)]
    env["PYTHONPATH"] = ROOT
    r = subprocess.run([sys.executable, "-m", "oracle.ref_bench"] + list(args), cwd=ROOT, env=env,
                       stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, timeout=timeout)
    if r.returncode != 0:
        raise RuntimeError(f"reference run failed: {r.stderr[-800:]}")
    return json.loads(r.stdout.strip().splitlines()[-1])


def available():
    return os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "site", "flowbench"))


def main():
    th = 1
    if "--threads" in sys.argv:
        th = int(sys.argv[sys.argv.index("--threads") + 1])
    for k, v in thread_env(th).items():  # before numpy / numba load their thread pools
        os.environ[k] = v
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["apply", "pcg"])
    ap.add_argument("--target", type=float, default=120_000)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--cases", default="cfg1,p4_16,p7_8")
    ap.add_argument("--threads", type=int, default=1)
    a = ap.parse_args()
    if a.what == "apply":
        res = apply_sweep(a.target, steps=a.steps, warmup=a.warmup, threads=a.threads)
    else:
        res = lor_pcg(a.cases.split(","))
    res["host_cpus"] = os.cpu_count()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
