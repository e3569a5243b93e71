"""Benchmark: fp64 GDoF/s of the sum-factorized 3D Helmholtz apply vs p.

Workload (BASELINE.json configs[1]): 3D Helmholtz
(c = 10, nu = 1; mass + diffusion) on a perturbed structured hex mesh of the
unit cube, ~10M DoFs for EVERY degree p = 1..8 (cfg2 shapes), quadrature
n_q = p + 2 Gauss-Legendre, stored quadrature-point factors (7 doubles per
point).  One step = one Helmholtz apply at each p = 1..8 (8 applies).
value = total DoFs processed / total device time (CUDA events, max over
ranks).  Per-degree GDoF/s and HBM-roofline fractions are reported in
`per_p`.  Every apply streams >= 1 GB of factors, far more than the 126 MB
L2, so no L2 flush is needed between iterations.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--impl reference` times the UNMODIFIED reference (flowbench 0.1.0, built into
oracle/_ref by oracle/build_ref.py) through its own HelmholtzOperator.apply,
numba backend, one thread, on a bounded sample of the same workload
(oracle/ref_bench.py, run as a subprocess: the product package is never
imported on that arm).  The GPU line's `cpu_baseline` and the LOR-PCG
reference solve times come from the same reference build, timed in the run.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEGREES = list(range(1, 9))
TARGET_DOFS = 10.0e6
C_HELM = 10.0
NU = 1.0
CPU_SAMPLE_DOFS = 120_000


def mesh_cells(p, target=TARGET_DOFS):
    return max(2, round((target ** (1.0 / 3.0) - 1.0) / p))


def algorithmic_bytes(N, ne, p, d=3, k=7):
    """read x + write y + int32 L->E map + stored factors."""
    return 16.0 * N + 4.0 * ne * (p + 1) ** d + 8.0 * k * ne * (p + 2) ** d


def algorithmic_flops(ne, p):
    """Optimal shared-intermediate count, Helmholtz."""
    n, q = p + 1, p + 2
    return ne * (2.0 * (4 * n ** 3 * q + 6 * n ** 2 * q ** 2 + 8 * n * q ** 3) + 17.0 * q ** 3)


def _traffic():
    """Measured DRAM bytes (read + write) of one sweep step -- every fused
    kernel and E->L sum launch -- from the committed ncu launch list
    (profiles/r2_traffic.json); None if the profile is absent."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r2_traffic.json")
    try:
        with open(path) as f:
            return int(json.load(f)["sweep_dram_bytes"])
    except (OSError, KeyError, ValueError):
        return None


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [s.strip() for s in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- problems

def build_problem(p, target=TARGET_DOFS, seed=1, rank=0, world=1):
    """One degree's problem.  world > 1: this rank's z-slab (n x n x n
    elements) of an n x n x (world*n) box, with a cut-plane halo exchange
    (weak scaling: ~target DoFs per GPU)."""
    from paper_1910_03032_b200 import geometry, mfop, partition, spaces
    n = mesh_cells(p, target)
    halo = None
    if world == 1:
        m = geometry.perturb_mesh(geometry.cartesian_mesh((n, n, n)), 0.05, seed=seed)
        sp = spaces.FESpace(m, p)
    else:
        slab = partition.StructuredSlab((n, n), n, p, rank, world, perturb=0.05, seed=seed)
        m, sp = slab.mesh, slab.space
        halo = partition.HaloExchange(slab, device="cuda")
    g = geometry.DeviceGeometry(m, sp.basis.quad)
    op = mfop.HelmholtzOperator(sp, g, C_HELM, nu=NU)
    ne = m.num_elements
    N = sp.ndofs
    del m
    return dict(p=p, n=n, ne=ne, N=N, op=op, halo=halo)


# ----------------------------------------------------------------------------- CPU legs

def cpu_problems(threads, target=CPU_SAMPLE_DOFS):
    """Oracle-port runners (reference apply restated in numpy) per degree."""
    from oracle import cpu_apply
    from paper_1910_03032_b200 import geometry, spaces
    out = []
    for p in DEGREES:
        n = mesh_cells(p, target)
        m = geometry.perturb_mesh(geometry.cartesian_mesh((n, n, n)), 0.05, seed=1)
        sp = spaces.FESpace(m, p)
        geom = geometry.compute_geometric_factors(m, sp.basis.quad)
        runner = cpu_apply.HelmholtzCPU(sp, geom, C_HELM, NU, threads=threads)
        x = np.random.default_rng(0).standard_normal(sp.ndofs)
        runner(x)  # warm
        out.append((runner, x, sp.ndofs))
    return out


def cpu_time(problems, reps=1):
    tot_dofs, tot_t = 0, 0.0
    for runner, x, n in problems:
        t0 = time.perf_counter()
        for _ in range(reps):
            runner(x)
        tot_t += time.perf_counter() - t0
        tot_dofs += reps * n
    return tot_dofs / tot_t / 1e9, tot_t


def run_reference(args, rank, world):
    """Reference arm: the UNMODIFIED reference (oracle/_ref, built from
    /root/reference by oracle/build_ref.py) timed through its own public API
    in a subprocess allowed every host thread (oracle/ref_bench.py; the
    reference's numba kernels are serial, so it uses one): stock
    HelmholtzOperator.apply, FLOWBENCH_BACKEND=numba, on a bounded sample of
    the workload.  Never imports the product package."""
    if rank != 0:
        return
    from oracle import ref_bench
    if ref_bench.available():
        res = ref_bench.run_subprocess(["apply", "--target", str(CPU_SAMPLE_DOFS),
                                        "--steps", str(args.steps), "--warmup", str(args.warmup)],
                                       threads=os.cpu_count() or 1)
        value, el, cores, kind, desc = (res["value"], res["seconds"], res["cores"], res["kind"],
                                        res["sample"])
        extra = {"per_p": res["per_p"], "host_cpus": res["host_cpus"], "setup_s": res["setup_s"]}
    else:  # no reference build on this host: the oracle port (test infrastructure)
        threads = os.cpu_count() or 1
        probs = cpu_problems(threads)
        for _ in range(args.warmup):
            cpu_time(probs)
        t0 = time.perf_counter()
        vals = [cpu_time(probs)[0] for _ in range(args.steps)]
        el = time.perf_counter() - t0
        for r, _, _ in probs:
            r.close()
        value, cores, kind = float(np.mean(vals)), threads, "port"
        desc = (f"3D Helmholtz apply, p=1..8, ~{CPU_SAMPLE_DOFS/1e3:.0f}k DoFs per degree, oracle "
                f"numpy port of the reference contractions on {threads} threads (oracle/_ref absent)")
        extra = {}
    cfg = config_block(world)
    cfg["sample_dofs_per_degree"] = CPU_SAMPLE_DOFS
    cfg["sample_note"] = ("the reference arm times a bounded sample (~120k DoFs per degree, "
                          "same mesh family, c, nu, quadrature) of the 10M-DoF-per-degree workload; "
                          "GDoF/s is size-normalised")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GDoF/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / max(args.steps, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": "GDoF/s", "cores": cores, "kind": kind,
                         "sample": desc},
        "e2e": {"value": value, "unit": "GDoF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    line.update(extra)
    print(json.dumps(line), flush=True)


def reference_cpu(what, args, timeout=1800):
    """The reference's own CPU path on this host (oracle/ref_bench.py), or
    an error note."""
    from oracle import ref_bench
    if not ref_bench.available():
        return {"error": "oracle/_ref not built (python oracle/build_ref.py)"}
    try:
        return ref_bench.run_subprocess([what] + list(args), timeout=timeout)
    except Exception as exc:  # the CPU leg must not drop the GPU line
        return {"error": f"{type(exc).__name__}: {exc}"[:300]}


PCG_CASES = {  # name -> (counts, p, kind, c); oracle/ref_bench.PCG_CASES
    "cfg1": ((16, 16), 4, "stiffness", 0.0),
    "p4_16": ((16, 16, 16), 4, "helmholtz", 10.0),
    "p7_8": ((8, 8, 8), 7, "helmholtz", 10.0),
    "p4_25": ((25, 25, 25), 4, "helmholtz", 10.0),
    "p7_14": ((14, 14, 14), 7, "helmholtz", 10.0),
}
REF_PCG_TIMED = ("cfg1", "p4_16", "p7_8")


def _golden_iterations():
    out = {"cfg1": 17}
    try:
        with open(os.path.join(ROOT, "tests", "golden", "manifest.json")) as f:
            man = json.load(f)
        for c in man.get("cfg3shape", []):
            if not c["perturb"]:
                out[f"p{c['p']}_{c['counts'][0]}"] = c["iterations"]
    except (OSError, KeyError, ValueError):
        pass
    return out


def lor_pcg(args, names=tuple(PCG_CASES)):
    """LOR-preconditioned CG time-to-solve on the device (parity mode:
    reference numbering, device operator + device V-cycle with the block
    ILU(0) smoother), rel_tol 1e-8, b = default_rng(0) normal with zero
    boundary values.  Beside it, the reference's own CPU solve
    of the same problem timed on this host in the same run (cases
    REF_PCG_TIMED; the ~1M-DoF cases carry the reference's golden counts)."""
    import torch
    from paper_1910_03032_b200 import geometry, mfop, solvers, spaces
    ref = reference_cpu("pcg", ["--cases", ",".join(REF_PCG_TIMED)]) if not args.no_cpu else {}
    gold = _golden_iterations()
    out = {}
    for name in names:
        counts, p, kind, c = PCG_CASES[name]
        t0 = time.perf_counter()
        m = geometry.cartesian_mesh(counts)
        sp = spaces.FESpace(m, p)
        geom = geometry.DeviceGeometry(m, sp.basis.quad)
        op = mfop.setup(kind, space=sp, geom=geom, nu=1.0, c=c)
        bdr = sp.boundary_dof_set()
        A = mfop.ConstrainedOperator(op, bdr)
        pre = solvers.LORPreconditioner(sp, kind, c=c, dirichlet_attrs="all")
        setup = time.perf_counter() - t0
        b = np.random.default_rng(0).standard_normal(sp.ndofs)
        b[bdr] = 0.0
        bd = torch.from_numpy(b).cuda()
        cfg = solvers.SolverConfig(rel_tol=1e-8, max_iters=300)
        solvers.cg(A, bd, precond=pre, config=cfg)  # warm
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        x, rep = solvers.cg(A, bd, precond=pre, config=cfg)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        ent = {"dofs": sp.ndofs, "iterations": rep.iterations, "converged": rep.converged,
               "solve_ms": round(ms, 2), "ms_per_iteration": round(ms / max(rep.iterations, 1), 3),
               "host_setup_s": round(setup, 2), "reference_iterations": gold.get(name)}
        r = ref.get(name) if isinstance(ref, dict) else None
        if r:
            ent["reference_cpu"] = {"iterations": r["iterations"], "solve_s": r["solve_s"],
                                    "setup_s": r["setup_s"], "cores": 1,
                                    "x_norm_rel_diff": abs(float(torch.linalg.norm(x)) - r["x_norm"])
                                    / r["x_norm"]}
            ent["speedup_solve"] = round(r["solve_s"] / (ms * 1e-3), 1)
        out[name] = ent
    if isinstance(ref, dict) and "error" in ref:
        out["reference_cpu_error"] = ref["error"]
    out["note"] = ("GPU: CUDA-event time of solvers.cg after one warm solve; reference_cpu: the "
                   "unmodified reference (oracle/_ref) cg + LORPreconditioner on this host, "
                   "FLOWBENCH_BACKEND=numba, 1 thread, same mesh / RHS")
    return out


def lor_pcg_scale(cases=((4, 116), (7, 66)), c=C_HELM):
    """cfg3 at full size (~100M DoFs, one GPU): scale-mode LOR-PCG with the
    whole hierarchy built on the device (structured.py: block-major numbering,
    device Q1 assembly, device block-ILU factor, matrix-free transfers,
    geometric Q1 coarsening).  Time-to-solve at rel_tol 1e-8 from CUDA events,
    plus the per-phase cost of one operator apply and one V-cycle."""
    import gc
    import torch
    from paper_1910_03032_b200 import solvers, structured as S
    out = {}
    for p, n in cases:
        t0 = time.perf_counter()
        prob = S.helmholtz_box_problem((n, n, n), p, c=c, perturb=0.05, seed=1)
        setup = time.perf_counter() - t0
        A, M, b = prob["A"], prob["M"], prob["b"]
        cfg = solvers.SolverConfig(rel_tol=1e-8, max_iters=300)
        solvers.cg(A, b, precond=M, config=cfg)  # warm
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        e[0].record()
        x, rep = solvers.cg(A, b, precond=M, config=cfg)
        e[1].record()
        y = torch.empty_like(b)
        e[2].record()
        A.apply_into(b, y)
        e[3].record()
        M.apply_into(b, y)
        e[4].record()
        torch.cuda.synchronize()
        ms = e[0].elapsed_time(e[1])
        N = prob["space"].ndofs_scalar
        peak, _ = load_peaks()
        lv = M.level_bytes()
        vbytes = sum(l["bytes"] for l in lv)
        vms = e[3].elapsed_time(e[4])
        ams = e[2].elapsed_time(e[3])
        abytes = algorithmic_bytes(N, prob["mesh"].num_elements, p)
        out[f"p{p}_{n}^3"] = {
            "dofs": N, "iterations": rep.iterations, "converged": rep.converged,
            "solve_ms": round(ms, 2), "ms_per_iteration": round(ms / max(rep.iterations, 1), 3),
            "apply_ms": round(ams, 3), "apply_hbm_frac": round(abytes / (ams * 1e-3) / 1e9 / peak, 4),
            "vcycle_ms": round(vms, 3), "vcycle_algorithmic_bytes": int(vbytes),
            "vcycle_hbm_frac": round(vbytes / (vms * 1e-3) / 1e9 / peak, 4),
            "vcycle_levels": [{k2: (int(v) if k2 != "kind" else v) for k2, v in l.items()}
                              for l in lv],
            "setup_s": round(setup, 2), "levels": M.describe(),
            "mode": "scale: block-ILU(2^3 elements) smoother, Q1 level coarsened "
                    "geometrically (near-exact: coarse_cycles stationary h-cycles) to a "
                    "dense-inverse bottom",
            "reference_iterations_1M": _golden_iterations().get({4: "p4_25", 7: "p7_14"}[p])}
        del prob, A, M, b, x, y
        gc.collect()
        torch.cuda.empty_cache()
    return out


def lor_pcg_sharded(rank, world, cases=((4, 116, 16, "weak"), (7, 66, 8, "weak"),
                                        (4, 116, 116, "strong"), (7, 68, 68, "strong")),
                    c=C_HELM):
    """cfg3 on N GPUs: scale-mode LOR-PCG sharded over z-slabs (dist_box.py).
    weak: `layers` element layers per rank on a (n, n, layers*N) box (p = 4:
    ~13.8M DoFs per GPU, 110M at 8 GPUs; p = 7: ~12M per GPU); strong: the
    fixed (n, n, nz) box split over the N ranks (116^3 p = 4: 100.5M DoFs, the
    single-GPU lor_pcg_cfg3 problem; 68^3 p = 7: 108.5M DoFs).  Time-to-solve
    from CUDA events between barriers, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_1910_03032_b200 import dist_box as D, solvers
    comm = D.TorchComm()
    out = {}
    for p, n, layers, mode in cases:
        counts = (n, n, layers * world) if mode == "weak" else (n, n, layers)
        t0 = time.perf_counter()
        pr = D.helmholtz_slab_problem(comm, counts, p, c=c, perturb=0.05, seed=1)
        setup = time.perf_counter() - t0
        cfg = solvers.SolverConfig(rel_tol=1e-8, max_iters=300)
        lv = pr["level"]
        D.dist_cg(pr["A"], pr["b"], pr["M"], comm, lv.n_own, cfg)  # warm
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x, rep = D.dist_cg(pr["A"], pr["b"], pr["M"], comm, lv.n_own, cfg)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ndofs = int(np.prod([a * p + 1 for a in counts]))
        out[f"{mode}_p{p}_{n}x{n}x{counts[2]}"] = {
            "dofs": ndofs, "dofs_per_gpu": ndofs // world, "iterations": rep.iterations,
            "converged": rep.converged, "solve_ms": round(float(t.item()), 2),
            "setup_s": round(setup, 2), "n_gpus": world, "scaling": mode,
            "note": "z-slab sharding: slab operator + NCCL halo sums, owned-row LOR levels, "
                    "slab block ILU, agglomerated Q1 V-cycle, all-reduced dots"}
        del pr, x
        import gc
        gc.collect()
        torch.cuda.empty_cache()
    return out


METRIC = "fp64 GDoF/s of sum-factorized Helmholtz apply vs p (3D, p=1..8, ~10M DoFs each)"


def callers(stokes_cases=((2, 2), (2, 4), (2, 6), (3, 2)), tgv=(5, 16, 4)):
    """Device time of the cfg4 / cfg5 callers: the
    lid-driven Stokes cavity by FGMRES with the block-triangular
    preconditioner (Taylor-Hood, rel_tol 1e-8; iteration counts beside the
    reference's from tests/golden/manifest.json), and projection steps of the
    periodic 3D Taylor-Green vortex (p, cells per direction, steps)."""
    import torch
    from paper_1910_03032_b200 import geometry, solvers, spaces, stokes, timeint
    man = {}
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "tests", "golden",
                               "manifest.json")) as f:
            man = {c["name"]: c for c in json.load(f).get("stokes", [])}
    except OSError:
        pass

    def lid(X):
        out = np.zeros_like(X)
        out[np.abs(X[:, 1] - 1.0) < 1e-12, 0] = 1.0
        return out

    out = {}
    for d, p in stokes_cases:
        counts = (8, 8) if d == 2 else (3, 3, 3)
        m = geometry.cartesian_mesh(counts)
        vs = spaces.FESpace(m, p, vdim=d)
        ps = spaces.FESpace(m, p - 1)
        geom = geometry.compute_geometric_factors(m, vs.basis.quad)
        t0 = time.perf_counter()
        S = stokes.StokesSystem(vs, ps, geom, nu=1.0)
        setup = time.perf_counter() - t0
        cfg = solvers.SolverConfig(rel_tol=1e-8, max_iters=200)
        S.solve(g=lid, config=cfg)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, _, rep = S.solve(g=lid, config=cfg)
        torch.cuda.synchronize()
        ms = 1e3 * (time.perf_counter() - t0)
        ref = man.get(f"cav{d}d_p{p}", {})
        out[f"stokes_cavity_{d}d_p{p}"] = {
            "dofs": int(vs.ndofs + ps.ndofs), "iterations": rep.iterations,
            "reference_iterations": ref.get("iterations"), "solve_ms": round(ms, 2),
            "setup_s": round(setup, 2), "timing": "host wall clock around StokesSystem.solve "
            "(host numpy in/out), after one warm-up solve"}
    p, n, steps = tgv
    m = geometry.cartesian_mesh((n, n, n), lows=(-np.pi,) * 3, highs=(np.pi,) * 3,
                                periodic=(True,) * 3)
    vs = spaces.FESpace(m, p, vdim=3)
    ps = spaces.FESpace(m, p)
    geom = geometry.compute_geometric_factors(m, vs.basis.quad)
    t0 = time.perf_counter()
    st = timeint.ProjectionStepper(vs, ps, geom, k=3, dt=0.02, nu=1.0 / 1600.0)

    def tgv_u(x):
        X, Y, Z = x[:, 0], x[:, 1], x[:, 2]
        return np.stack([np.sin(X) * np.cos(Y) * np.cos(Z), -np.cos(X) * np.sin(Y) * np.cos(Z),
                         np.zeros_like(X)], axis=1)

    st.initialize(vs.project(tgv_u))
    for _ in range(3):  # BDF1..3 start-up: each new order builds its Helmholtz LOR hierarchy
        st.step()
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    its = []
    t0 = time.perf_counter()
    for _ in range(steps):
        r = st.step()
        its.append([r.mass_iters, r.pressure_iters, r.helmholtz_iters])
    torch.cuda.synchronize()
    ms = 1e3 * (time.perf_counter() - t0) / steps
    st.profile = True  # one more step with CUDA events between its phases
    phases = st.step().phase_ms
    st.profile = False
    out[f"tgv3d_projection_p{p}_{n}^3"] = {
        "velocity_dofs": int(vs.ndofs), "pressure_dofs": int(ps.ndofs), "ms_per_step": round(ms, 2),
        "steps": steps, "iterations_mass_pressure_helmholtz": its, "setup_s": round(setup, 2),
        "phase_ms": phases,
        "kinetic_energy": st.kinetic_energy(),
        "scheme": "BDF3/EXT3, dt 0.02, nu 1/1600; timed after the 3 start-up steps (setup_s)"}
    del st
    out.update(box_tgv(p=p, n=32, steps=2))
    return out


def box_tgv(p=5, n=32, steps=2):
    """cfg5 at size on one GPU: the periodic Taylor-Green projection in scale
    mode (timeint.BoxProjectionStepper: BoxSpace numbering, device-built
    pure-Neumann / Helmholtz block-ILU hierarchies), n^3 elements."""
    import gc
    import torch
    from paper_1910_03032_b200 import geometry, timeint
    gc.collect()
    torch.cuda.empty_cache()
    m = geometry.cartesian_mesh((n, n, n), lows=(-np.pi,) * 3, highs=(np.pi,) * 3,
                                periodic=(True,) * 3)
    t0 = time.perf_counter()
    st = timeint.BoxProjectionStepper(m, p, k=3, dt=0.02, nu=1.0 / 1600.0)

    def tgv_u(x):
        X, Y, Z = x[:, 0], x[:, 1], x[:, 2]
        return np.stack([np.sin(X) * np.cos(Y) * np.cos(Z), -np.cos(X) * np.sin(Y) * np.cos(Z),
                         np.zeros_like(X)], axis=1)

    st.initialize(st.vspace.project(tgv_u))
    for _ in range(3):
        st.step()
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    its = []
    t0 = time.perf_counter()
    for _ in range(steps):
        r = st.step()
        its.append([r.mass_iters, r.pressure_iters, r.helmholtz_iters])
    torch.cuda.synchronize()
    ms = 1e3 * (time.perf_counter() - t0) / steps
    st.profile = True
    phases = st.step().phase_ms
    res = {f"tgv3d_projection_scale_mode_p{p}_{n}^3": {
        "velocity_dofs": int(st.vspace.ndofs), "pressure_dofs": int(st.pspace.ndofs),
        "ms_per_step": round(ms, 2), "steps": steps, "iterations_mass_pressure_helmholtz": its,
        "setup_s": round(setup, 2), "phase_ms": phases, "kinetic_energy": st.kinetic_energy(),
        "scheme": "BDF3/EXT3, dt 0.02, nu 1/1600, scale mode (BoxProjectionStepper)"}}
    del st
    gc.collect()
    torch.cuda.empty_cache()
    return res


def _max_over_ranks(v):
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def box_tgv_sharded(comm, p=5, n=64, steps=2, reduce_max=None):
    """cfg5 on N GPUs: the periodic Taylor-Green projection step sharded over
    z-slabs on a ring (dist_periodic.DistProjectionStepper), strong scaling of
    the n^3 box (64^3 p = 5: 98.3M velocity + 32.8M pressure DoFs; 16 slab
    units of 4 layers, balanced on 2, 4 and 8 ranks).  Per-step time from CUDA
    events between barriers; reduce_max(ms) -> max over ranks (NCCL
    all-reduce in the bench)."""
    import gc
    import torch
    from paper_1910_03032_b200 import dist_periodic as DP, geometry
    gc.collect()
    torch.cuda.empty_cache()
    m = geometry.cartesian_mesh((n, n, n), lows=(-np.pi,) * 3, highs=(np.pi,) * 3,
                                periodic=(True,) * 3)
    t0 = time.perf_counter()
    st = DP.DistProjectionStepper(comm, m, p, k=3, dt=0.02, nu=1.0 / 1600.0)

    def tgv_u(x):
        X, Y, Z = x[:, 0], x[:, 1], x[:, 2]
        return np.stack([np.sin(X) * np.cos(Y) * np.cos(Z), -np.cos(X) * np.sin(Y) * np.cos(Z),
                         np.zeros_like(X)], axis=1)

    st.initialize_from(tgv_u)
    for _ in range(3):
        st.step()
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    its = []
    comm.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        r = st.step()
        its.append([r.mass_iters, r.pressure_iters, r.helmholtz_iters])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if reduce_max is not None:
        ms = reduce_max(ms)
    energy = st.kinetic_energy()
    res = {f"tgv3d_projection_ring_p{p}_{n}^3": {
        "velocity_dofs": 3 * (n * p) ** 3, "pressure_dofs": (n * p) ** 3,
        "ms_per_step": round(ms, 2), "steps": steps, "iterations_mass_pressure_helmholtz": its,
        "setup_s": round(setup, 2), "kinetic_energy": energy, "n_gpus": comm.world,
        "scaling": "strong", "layers_per_rank": [b - a for a, b in st.layers],
        "scheme": "BDF3/EXT3, dt 0.02, nu 1/1600; z-slabs on a periodic ring "
                  "(dist_periodic.DistProjectionStepper), ring halos over NCCL"}}
    del st
    gc.collect()
    torch.cuda.empty_cache()
    return res


def mixed_and_vector_ops(reps=10, target=TARGET_DOFS / 3):
    """Device time and HBM-roofline fraction of the Stokes / projection
    blocks: the fused mixed-degree kernel's G, G^T, D and
    the vdim = 3 vector Laplacian, on perturbed cubes with ~`target` DoFs per
    velocity component (cfg4 Taylor-Hood p=4/3, cfg5 equal order p=5).
    Algorithmic bytes (k = d^2 = 9 for G/D): input + output
    vectors + int32 maps of both spaces + stored factors."""
    import torch
    from paper_1910_03032_b200 import _lib, geometry, mfop, spaces
    peak, _ = load_peaks()
    out = {}
    for pv, pp in ((4, 3), (5, 5)):
        n = mesh_cells(pv, target)
        m = geometry.perturb_mesh(geometry.cartesian_mesh((n, n, n)), 0.05, seed=1)
        vs = spaces.FESpace(m, pv, vdim=3)
        ps = spaces.FESpace(m, pp)
        g = geometry.DeviceGeometry(m, vs.basis.quad)
        ne, q3 = m.num_elements, (pv + 2) ** 3
        nv, npd = vs.ndofs_scalar, ps.ndofs_scalar
        G = mfop.GradientOperator(vs, ps, g)
        D = mfop.DivergenceOperator(vs, ps, g)
        L = mfop.StiffnessOperator(vs, g)
        maps = 4.0 * ne * ((pv + 1) ** 3 + (pp + 1) ** 3)
        cases = {
            "G": (lambda a, b: G.apply_into(a, b), npd, 3 * nv,
                  8.0 * (npd + 3 * nv) + maps + 72.0 * ne * q3),
            "Gt": (lambda a, b: G.apply_transpose_into(a, b), 3 * nv, npd,
                   8.0 * (npd + 3 * nv) + maps + 72.0 * ne * q3),
            "D": (lambda a, b: D.apply_into(a, b), 3 * nv, npd,
                  8.0 * (npd + 3 * nv) + maps + 72.0 * ne * q3),
            "vector_laplacian": (lambda a, b: L.apply_into(a, b), 3 * nv, 3 * nv,
                                 48.0 * nv + 4.0 * ne * (pv + 1) ** 3 + 48.0 * ne * q3),
        }
        res = {"velocity_dofs": 3 * nv, "pressure_dofs": npd, "elements": ne,
               "fused_mixed": bool(_lib.lib.fb_operator_fast_path(G.handle) == 2)}
        for name, (fn, nin, nout, by) in cases.items():
            xa = torch.randn(nin, dtype=torch.float64, device="cuda")
            ya = torch.empty(nout, dtype=torch.float64, device="cuda")
            for _ in range(3):
                fn(xa, ya)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                fn(xa, ya)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            res[name] = {"ms": round(ms, 4), "gdofs_in_plus_out": round((nin + nout) / ms / 1e6, 3),
                         "hbm_frac": round(by / (ms * 1e-3) / 1e9 / peak, 4),
                         "algorithmic_bytes": int(by)}
        out[f"3d_pv{pv}_pp{pp}"] = res
        del G, D, L, g
    return out


def config_block(world):
    return {"workload": "cfg2-shape 3D Helmholtz apply sweep p=1..8, ~10M DoFs per degree, "
                        "perturbed unit-cube hex mesh, n_q=p+2 Gauss-Legendre, stored factors",
            "c": C_HELM, "nu": NU, "degrees": DEGREES, "target_dofs_per_degree": TARGET_DOFS,
            "parallelism": (f"z-slab x{world} (weak scaling: n x n x n elements per GPU, "
                            f"NCCL cut-plane halo sum per apply)") if world > 1 else "single GPU",
            "l2_policy": "per-apply working set >= 1 GB (factors) >> 126 MB L2; no flush needed"}


# ----------------------------------------------------------------------------- GPU leg

def run_ours(args, rank, world):
    import torch
    import torch.distributed as dist
    from paper_1910_03032_b200 import _lib

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    probs = [build_problem(p, rank=rank, world=world) for p in DEGREES]
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    for pr in probs:
        pr["x"] = torch.randn(pr["N"], dtype=torch.float64, device="cuda", generator=gen)
        pr["y"] = torch.empty_like(pr["x"])
    st = torch.cuda.current_stream()

    def step(timed_events=None):
        for i, pr in enumerate(probs):
            if timed_events is not None:
                timed_events[i][0].record(st)
            pr["op"].apply_into(pr["x"], pr["y"])
            if pr["halo"] is not None:
                pr["halo"].sum(pr["y"])
            if timed_events is not None:
                timed_events[i][1].record(st)

    clocks = ClockSampler(local)
    clocks.start()
    tw = time.perf_counter()
    nw = 0
    while nw < args.warmup or time.perf_counter() - tw < 1.0:  # >= W warm-up steps, >= 1 s loaded
        step()
        nw += 1
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in probs] for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    l0 = _lib.lib.fb_launch_count()
    torch.cuda.synchronize()
    t_start.record(st)
    for k in range(args.steps):
        step(evs[k])
    t_end.record(st)
    torch.cuda.synchronize()
    launches = _lib.lib.fb_launch_count() - l0
    clk = clocks.stop()
    total_ms = t_start.elapsed_time(t_end)
    per_p_ms = [float(np.mean([evs[k][i][0].elapsed_time(evs[k][i][1])
                               for k in range(args.steps)])) for i in range(len(probs))]
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())

    # kernel-level timing of the fused element kernel alone (part 1), per p
    kern_ms = []
    for pr in probs:
        op = pr["op"]
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        reps = 5
        a.record(st)
        for _ in range(reps):
            _lib.check(_lib.lib.fb_operator_apply_part(op.handle, pr["x"].data_ptr(),
                                                       pr["y"].data_ptr(), 1, st.cuda_stream))
        b.record(st)
        torch.cuda.synchronize()
        kern_ms.append(a.elapsed_time(b) / reps)

    # e2e through the public API with pinned host buffers, copies timed.
    # Three streams pipeline the sweep: H2D of degree i+1 and D2H of degree
    # i-1 overlap the apply of degree i (PCIe is full duplex); events keep
    # the per-degree buffers' hazards across steps.
    hx = [torch.empty(pr["N"], dtype=torch.float64, pin_memory=True) for pr in probs]
    hy = [torch.empty(pr["N"], dtype=torch.float64, pin_memory=True) for pr in probs]
    for h, pr in zip(hx, probs):
        h.copy_(pr["x"].cpu())
    e2e_steps = max(1, min(args.steps, 5))
    s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event()  # noqa: E731
    done_in = [ev() for _ in probs]
    done_cmp = [ev() for _ in probs]
    done_out = [ev() for _ in probs]
    first = [True]

    def e2e_step():
        for i, pr in enumerate(probs):
            with torch.cuda.stream(s_in):
                if not first[0]:
                    s_in.wait_event(done_cmp[i])  # x_i consumed by the previous step
                pr["x"].copy_(hx[i], non_blocking=True)
                done_in[i].record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(done_in[i])
                if not first[0]:
                    s_cmp.wait_event(done_out[i])  # y_i read back by the previous step
                pr["op"].apply_into(pr["x"], pr["y"])
                if pr["halo"] is not None:
                    pr["halo"].sum(pr["y"])
                done_cmp[i].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(done_cmp[i])
                hy[i].copy_(pr["y"], non_blocking=True)
                done_out[i].record(s_out)
        first[0] = False

    e2e_step()
    torch.cuda.synchronize()
    ea = torch.cuda.Event(enable_timing=True)
    eb = torch.cuda.Event(enable_timing=True)
    ea.record(s_in)
    s_cmp.wait_event(ea)
    s_out.wait_event(ea)
    for _ in range(e2e_steps):
        e2e_step()
    tail_in, tail_cmp = torch.cuda.Event(), torch.cuda.Event()
    tail_in.record(s_in)
    tail_cmp.record(s_cmp)
    s_out.wait_event(tail_in)
    s_out.wait_event(tail_cmp)
    eb.record(s_out)
    torch.cuda.synchronize()
    e2e_ms = ea.elapsed_time(eb) / e2e_steps
    ok = all(torch.equal(hy[i], pr["y"].cpu()) for i, pr in enumerate(probs))

    # the same copies with the applies removed, H2D and D2H streams independent
    # (full duplex): the PCIe bound of the e2e figure on this box (hosts differ
    # in link / NUMA placement from box to box)
    def copy_step():
        for i, pr in enumerate(probs):
            with torch.cuda.stream(s_in):
                pr["x"].copy_(hx[i], non_blocking=True)
                done_in[i].record(s_in)
            with torch.cuda.stream(s_out):
                hy[i].copy_(pr["y"], non_blocking=True)

    copy_step()
    torch.cuda.synchronize()
    ea.record(s_in)
    s_out.wait_event(ea)
    for _ in range(e2e_steps):
        copy_step()
    tail_in.record(s_in)
    s_out.wait_event(tail_in)
    eb.record(s_out)
    torch.cuda.synchronize()
    copy_ms = ea.elapsed_time(eb) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # the drop-in call a reference user makes: op.apply(numpy array) per degree
    # (pageable input arrays; synchronous H2D / apply / D2H through cached pinned
    # blocks; no pipelining)
    xh = [h.numpy().copy() for h in hx]  # ordinary (pageable) user arrays
    for pr, xv in zip(probs, xh):
        pr["op"].apply(xv)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for pr, xv in zip(probs, xh):
        pr["op"].apply(xv)
    torch.cuda.synchronize()
    numpy_ms = 1e3 * (time.perf_counter() - t0)

    sharded = None
    meta = [{"N": pr["N"], "ne": pr["ne"], "p": pr["p"], "fast": pr["op"].fast_path}
            for pr in probs]
    if world > 1 and not args.no_cfg3:
        import gc
        probs.clear()
        gc.collect()
        torch.cuda.empty_cache()
        try:
            sharded = lor_pcg_sharded(rank, world)
        except Exception as exc:  # keep the headline line if the auxiliary solve fails
            sharded = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        if not args.no_callers:
            try:
                from paper_1910_03032_b200 import dist_box as D
                sharded.update(box_tgv_sharded(D.TorchComm(), reduce_max=_max_over_ranks))
            except Exception as exc:
                sharded["tgv_error"] = f"{type(exc).__name__}: {exc}"[:300]
    if rank != 0:
        return
    peak, peak_kind = load_peaks()
    dofs_step = float(sum(m["N"] for m in meta))
    ms_step = total_ms / args.steps
    value = world * dofs_step / (ms_step * 1e-3) / 1e9
    per_p = {}
    tot_bytes = 0.0
    for pr, ms, kms in zip(meta, per_p_ms, kern_ms):
        by = algorithmic_bytes(pr["N"], pr["ne"], pr["p"])
        tot_bytes += by
        per_p[str(pr["p"])] = {
            "dofs": pr["N"], "elements": pr["ne"], "ms": round(ms, 4),
            "gdofs": round(pr["N"] / (ms * 1e-3) / 1e9, 3),
            "hbm_frac": round(by / (ms * 1e-3) / 1e9 / peak, 4),
            "kernel_ms": round(kms, 4),
            "kernel_hbm_frac": round(by / (kms * 1e-3) / 1e9 / peak, 4),
            "tflops": round(algorithmic_flops(pr["ne"], pr["p"]) / (ms * 1e-3) / 1e12, 2),
            "fast_path": pr["fast"],
        }
    achieved = tot_bytes / (sum(per_p_ms) * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "GDoF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_block(world),
        "per_p": per_p,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": _traffic(), "algorithmic_bytes_per_step": int(tot_bytes),
                     "peak_source": peak_kind,
                     "note": "full apply (fused element kernel + E->L sum of shared DoFs), "
                             "algorithmic bytes 16N + 4 ne (p+1)^3 + 56 ne (p+2)^3 over the "
                             "p=1..8 sweep"},
        "e2e": {"value": round(world * dofs_step / (e2e_ms * 1e-3) / 1e9, 4), "unit": "GDoF/s",
                "h2d_bytes_per_step": int(8 * dofs_step), "d2h_bytes_per_step": int(8 * dofs_step),
                "note": "HelmholtzOperator.apply_into per degree, pinned-host x/y copies inside "
                        "the timed region, H2D/apply/D2H pipelined over the sweep on 3 streams",
                "readback_matches_device": ok,
                "copy_only": {"ms_per_step": round(copy_ms, 3),
                              "gdofs": round(world * dofs_step / (copy_ms * 1e-3) / 1e9, 4),
                              "gbps_per_direction": round(8 * dofs_step / (copy_ms * 1e-3) / 1e9,
                                                          1),
                              "note": "same pinned H2D/D2H copies, applies removed: the "
                                      "PCIe bound of this box"},
                "numpy_api": {"value": round(world * dofs_step / (numpy_ms * 1e-3) / 1e9, 4),
                              "unit": "GDoF/s",
                              "note": "HelmholtzOperator.apply(numpy) per degree on ordinary "
                                      "(pageable) numpy inputs, synchronous; operand and "
                                      "result cross through cached pinned host blocks "
                                      "(device.to_device / to_host); host wall clock, one "
                                      "sweep"}},
        "gpu_launches": int(launches),
        "clocks": clk,
        "warmup_steps_run": nw,
    }
    if not args.no_pcg and world == 1:
        line["lor_pcg"] = lor_pcg(args)
    if sharded is not None:
        line["lor_pcg_cfg3_sharded"] = sharded
    if not args.no_callers and world == 1:
        try:
            line["mixed_and_vector_ops"] = mixed_and_vector_ops()
        except Exception as exc:
            line["mixed_and_vector_ops"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        try:
            line["callers"] = callers()
        except Exception as exc:  # a caller failure must not drop the headline line
            line["callers"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    if not args.no_cfg3 and world == 1:
        import gc
        import torch
        probs.clear()
        gc.collect()
        torch.cuda.empty_cache()
        line["lor_pcg_cfg3"] = lor_pcg_scale()
    if not args.no_cpu:
        res = reference_cpu("apply", ["--target", str(CPU_SAMPLE_DOFS), "--steps", "2",
                                      "--warmup", "1"])
        if "error" not in res:
            line["cpu_baseline"] = {"value": res["value"], "unit": "GDoF/s", "cores": res["cores"],
                                    "kind": res["kind"], "sample": res["sample"],
                                    "seconds": round(res["seconds"], 2),
                                    "host_cpus": res["host_cpus"], "per_p": res["per_p"]}
        else:
            line["cpu_baseline"] = res
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-pcg", action="store_true")
    ap.add_argument("--no-cfg3", action="store_true", help="skip the 100M-DoF LOR-PCG solves")
    ap.add_argument("--no-callers", action="store_true", help="skip the cfg4/cfg5 caller timings")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # the driver's log shows the NCCL transport
        dist.init_process_group("nccl")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world)
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
