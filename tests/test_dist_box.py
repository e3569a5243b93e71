"""Sharded scale mode (paper_1910_03032_b200/dist_box.py).

The multi-rank path runs as R threads of one process on one GPU through the
in-process communicator (host-side barriers only; no kernel waits on another
rank), so the NCCL code path's algorithm -- slab layout, halo exchanges,
owned-slice dots, agglomerated Q1 solve -- is checked against the single-GPU
scale-mode solve on the same global problem."""

import numpy as np
import pytest

from tests.cases import rel_err


def test_slab_layers_align_to_units():
    from paper_1910_03032_b200 import dist_box as D
    assert D.slab_layers(12, 3, 4) == [(0, 4), (4, 8), (8, 12)]
    assert D.slab_layers(16, 3, 4) == [(0, 4), (4, 8), (8, 16)]
    with pytest.raises(ValueError):
        D.slab_layers(10, 2, 4)
    with pytest.raises(ValueError):
        D.slab_layers(8, 3, 4)


def test_thread_comm_exchange_and_reductions():
    import torch
    from paper_1910_03032_b200 import dist_box as D

    def fn(comm):
        r, w = comm.rank, comm.world
        sd = torch.full((3,), float(10 * r + 1)) if r > 0 else None
        su = torch.full((3,), float(10 * r + 2)) if r < w - 1 else None
        rd = torch.empty(3) if r > 0 else None
        ru = torch.empty(3) if r < w - 1 else None
        comm.exchange(sd, su, rd, ru)
        s = comm.allreduce_sum(torch.tensor([float(r + 1)]))
        g = comm.allgather(torch.arange(r + 1, dtype=torch.float64), list(range(1, w + 1)))
        return (None if rd is None else rd[0].item(), None if ru is None else ru[0].item(),
                s.item(), g.tolist())

    import unittest.mock as um
    with um.patch.object(torch.cuda, "synchronize", lambda: None):
        out = D.run_threads(3, fn)
    assert out[0][:2] == (None, 11.0) and out[1][:2] == (2.0, 21.0) and out[2][:2] == (12.0, None)
    assert all(o[2] == 6.0 for o in out)
    assert out[0][3] == [0.0, 0.0, 1.0, 0.0, 1.0, 2.0]


def _torchcomm_worker(rank, world, port, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1910_03032_b200 import dist_box as D
        comm = D.TorchComm()
        r, w = comm.rank, comm.world
        sd = torch.full((3,), float(10 * r + 1)) if r > 0 else None
        su = torch.full((3,), float(10 * r + 2)) if r < w - 1 else None
        rd = torch.empty(3) if r > 0 else None
        ru = torch.empty(3) if r < w - 1 else None
        comm.exchange(sd, su, rd, ru)
        s = comm.allreduce_sum(torch.tensor([float(r + 1)], dtype=torch.float64))
        g = comm.allgather(torch.arange(r + 1, dtype=torch.float64), list(range(1, w + 1)))
        # periodic ring: every rank exchanges with both neighbours (mod world)
        ring_d, ring_u = torch.empty(3), torch.empty(3)
        comm.exchange_ring(torch.full((3,), float(10 * r + 1)), torch.full((3,), float(10 * r + 2)),
                           ring_d, ring_u)
        q.put((r, None if rd is None else rd[0].item(), None if ru is None else ru[0].item(),
               s.item(), g.tolist(), ring_d[0].item(), ring_u[0].item()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_torch_comm_over_gloo_matches_thread_comm(world):
    """The torch.distributed communicator (NCCL on the GPU box) has the
    same exchange / ring exchange / all-reduce / all-gather semantics (gloo,
    2 and 3 processes; on 2 ranks both ring neighbours are the same peer)."""
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_torchcomm_worker, args=(r, world, port, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    out = sorted(q.get(timeout=240) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    if world == 3:
        assert out[0][1:3] == (None, 11.0) and out[1][1:3] == (2.0, 21.0)
        assert out[2][1:3] == (12.0, None)
    else:
        assert out[0][1:3] == (None, 11.0) and out[1][1:3] == (2.0, None)
    assert all(o[3] == world * (world + 1) / 2 for o in out)
    gather = [float(j) for i in range(1, world + 1) for j in range(i)]
    assert all(o[4] == gather for o in out)
    for r, o in enumerate(out):
        assert o[5] == 10 * ((r - 1) % world) + 2  # from the lower neighbour's up-send
        assert o[6] == 10 * ((r + 1) % world) + 1  # from the upper neighbour's down-send


@pytest.mark.gpu
@pytest.mark.parametrize("world,counts,p,dq1", [(2, (3, 4, 8), 4, True), (3, (4, 3, 12), 2, True),
                                               (2, (2, 3, 8), 7, True), (2, (3, 4, 8), 4, False),
                                               (3, (4, 4, 12), 3, True)])
def test_sharded_lor_pcg_matches_single_gpu(world, counts, p, dq1):
    """cfg3 on N ranks: the Q1 level is sharded too (dq1: its stationary
    cycles on the slabs, the h-coarse box agglomerated) or agglomerated whole."""
    import torch
    from paper_1910_03032_b200 import dist_box as D, solvers, structured as S
    cfg = solvers.SolverConfig(rel_tol=1e-8, max_iters=300)
    mesh = S.box_mesh(counts, perturb=0.05, seed=1)
    ref = S.helmholtz_box_problem(counts, p, c=10.0, max_coarse=100)
    x_ref, rep_ref = solvers.cg(ref["A"], ref["b"], precond=ref["M"], config=cfg)
    x_ref = x_ref.cpu().numpy()
    y_ref = ref["A"].apply(ref["b"]).cpu().numpy()

    def fn(comm):
        pr = D.helmholtz_slab_problem(comm, counts, p, c=10.0, max_coarse=100, mesh=mesh,
                                      distribute_q1=dq1)
        assert pr["M"].q1_sharded == dq1
        lv = pr["level"]
        y = torch.empty_like(pr["b"])
        pr["A"].apply_into(pr["b"], y)
        x, rep = D.dist_cg(pr["A"], pr["b"], pr["M"], comm, lv.n_own, cfg)
        return lv.off, lv.n_own, y[:lv.n_own].cpu().numpy(), x[:lv.n_own].cpu().numpy(), rep

    out = D.run_threads(world, fn)
    assert [o[0] for o in out] == list(np.cumsum([0] + [o[1] for o in out[:-1]]))
    y = np.concatenate([o[2] for o in out])
    x = np.concatenate([o[3] for o in out])
    assert rel_err(y, y_ref) < 1e-13
    for o in out:
        assert o[4].iterations == out[0][4].iterations
    assert out[0][4].iterations == rep_ref.iterations, (out[0][4].iterations,
                                                        rep_ref.iterations)
    assert rel_err(x, x_ref) < 1e-7


@pytest.mark.gpu
@pytest.mark.parametrize("world,counts,p,kind", [(2, (4, 6, 8), 3, "stiffness"),
                                                  (3, (6, 4, 12), 5, "stiffness"),
                                                  (2, (6, 6, 8), 4, "helmholtz")])
def test_periodic_ring_lor_pcg_matches_single_gpu(world, counts, p, kind):
    """cfg5 building block on N ranks: periodic [-pi, pi]^3 box sharded into
    z-slabs on a ring (dist_periodic.py).  The sharded operator equals the
    single-GPU BoxSpace operator; the pure-Neumann Poisson solve (pinned
    levels, mean projection) or the Helmholtz solve gives the single-GPU
    scale-mode iteration count and solution."""
    import torch
    from paper_1910_03032_b200 import dist_box as D, dist_periodic as DP, geometry, mfop
    from paper_1910_03032_b200 import solvers, structured as S
    pn = kind == "stiffness"
    c = 0.0 if pn else 10.0
    cfg = solvers.SolverConfig(rel_tol=1e-10 if pn else 1e-8, max_iters=300)
    mesh = geometry.cartesian_mesh(counts, lows=(-np.pi,) * 3, highs=(np.pi,) * 3,
                                   periodic=(True,) * 3)
    space = S.BoxSpace(mesh, p, block=2, device=torch.device("cuda"))
    op = mfop.setup(kind, space=space, geom=geometry.DeviceGeometry(mesh, space.basis.quad),
                    nu=1.0, c=c)
    if pn:
        pre = S.BoxLORPreconditioner(space, kind, dirichlet_attrs=None, pure_neumann=True)
    else:
        pre = S.BoxLORPreconditioner(space, kind, nu=1.0, c=c)

    def fn(comm):
        pr = DP.periodic_slab_problem(comm, counts, p, kind=kind, c=c, pure_neumann=pn, mesh=mesh)
        lv = pr["level"]
        y = torch.empty_like(pr["b"])
        pr["A"].apply_into(pr["b"], y)
        x, rep = DP.dist_cg(pr["A"], pr["b"], pr["M"], comm, lv.n_own, cfg, project=pr["project"])
        return (lv.off, lv.n_own, y[:lv.n_own].cpu().numpy(), x[:lv.n_own].cpu().numpy(), rep,
                pr["b_global"].cpu().numpy())

    out = D.run_threads(world, fn)
    bg = torch.from_numpy(out[0][5]).cuda()
    y_ref = op.apply(bg).cpu().numpy()
    x_ref, rep_ref = solvers.cg(op, bg, precond=pre, config=cfg,
                                project=solvers.MeanProjector() if pn else None)
    x_ref = x_ref.cpu().numpy()
    assert [o[0] for o in out] == list(np.cumsum([0] + [o[1] for o in out[:-1]]))
    y = np.concatenate([o[2] for o in out])
    x = np.concatenate([o[3] for o in out])
    assert rel_err(y, y_ref) < 1e-13
    for o in out:
        assert o[4].iterations == out[0][4].iterations and o[4].converged
    assert out[0][4].iterations == rep_ref.iterations, (out[0][4].iterations,
                                                        rep_ref.iterations)
    assert rel_err(x, x_ref) < 1e-7


@pytest.mark.gpu
@pytest.mark.parametrize("world,counts,p", [(2, (4, 4, 8), 3), (3, (4, 6, 12), 2)])
def test_ring_projection_stepper_matches_single_gpu(world, counts, p):
    """cfg5 on N ranks: the periodic Taylor-Green projection step sharded
    over a ring of z-slabs (dist_periodic.DistProjectionStepper) against the
    single-GPU scale-mode stepper (timeint.BoxProjectionStepper, itself pinned
    to the reference golden): sub-solve counts +-1, velocity and energy."""
    from paper_1910_03032_b200 import dist_box as D, dist_periodic as DP, geometry, timeint
    mesh = geometry.cartesian_mesh(counts, lows=(-np.pi,) * 3, highs=(np.pi,) * 3,
                                   periodic=(True,) * 3)

    def tgv(x):
        X, Y, Z = x[:, 0], x[:, 1], x[:, 2]
        return np.stack([np.sin(X) * np.cos(Y) * np.cos(Z), -np.cos(X) * np.sin(Y) * np.cos(Z),
                         np.zeros_like(X)], axis=1)

    one = timeint.BoxProjectionStepper(mesh, p, k=3, dt=0.02, nu=1.0 / 1600.0)
    u0 = one.vspace.project(tgv)
    one.initialize(u0)
    ref_its = []
    for _ in range(4):
        r = one.step()
        ref_its.append([r.mass_iters, r.pressure_iters, r.helmholtz_iters])
    u_ref = one.u.cpu().numpy()
    e_ref = one.kinetic_energy()

    def fn(comm):
        st = DP.DistProjectionStepper(comm, mesh, p, k=3, dt=0.02, nu=1.0 / 1600.0)
        st.initialize_from(tgv)
        u_local = st.u.clone()
        st.initialize(u0)
        assert rel_err(u_local.cpu().numpy(), st.u.cpu().numpy()) < 1e-14
        its = []
        for _ in range(4):
            r = st.step()
            its.append([r.mass_iters, r.pressure_iters, r.helmholtz_iters])
        parts = st.gather_owned(st.u, 3)
        return its, np.concatenate([q.cpu().numpy() for q in parts]), st.kinetic_energy()

    out = D.run_threads(world, fn)
    for its, u, e in out:
        assert its == out[0][0]
        assert its == ref_its, (its, ref_its)  # the same V-cycles: equal counts
        assert rel_err(u, u_ref) < 1e-8
        assert e == pytest.approx(e_ref, rel=1e-10)


@pytest.mark.parametrize("world,counts,p", [(2, (4, 4, 8), 3), (3, (4, 6, 12), 2), (3, (3, 4, 12), 4)])
def test_periodic_ring_layout_host(world, counts, p):
    """Host logic of the periodic ring (no GPU): owned slices partition the
    global box numbering in rank order; every rank's element map, pulled back
    to global ids through [owned | lower ghost | upper ghost], is the global
    BoxSpace element map of its elements; each ghost plane is exactly what
    the neighbour around the ring sends."""
    import torch
    from paper_1910_03032_b200 import dist_box as D, dist_periodic as DP, geometry, structured as S
    cpu = torch.device("cpu")
    m = geometry.cartesian_mesh(counts, lows=(-np.pi,) * 3, highs=(np.pi,) * 3,
                                periodic=(True,) * 3)
    g = S.BoxSpace(m, p, block=2, device=cpu)
    ged = np.asarray(g.element_dofs)
    layers = D.slab_layers(counts[2], world, 4)
    lvs = [DP.PeriodicSlabLevel(m, p, 2, layers, r, world, cpu) for r in range(world)]
    assert [lv.off for lv in lvs] == list(np.cumsum([0] + [lv.n_own for lv in lvs[:-1]]))
    assert lvs[-1].off + lvs[-1].n_own == g.ndofs
    ne_layer = counts[0] * counts[1]
    for r, lv in enumerate(lvs):
        l2g = np.concatenate([np.arange(lv.off, lv.off + lv.n_own),
                              lv.ghost_gids["lower"].numpy(), lv.ghost_gids["upper"].numpy()])
        assert l2g.shape[0] == lv.n_local
        led = np.asarray(lv.element_dofs)
        e0, e1 = layers[r]
        assert np.array_equal(l2g[led], ged[e0 * ne_layer:e1 * ne_layer])
        down, up = lvs[(r - 1) % world], lvs[(r + 1) % world]
        # lower ghost <- the lower neighbour's up-send; upper ghost <- the upper's down-send
        assert np.array_equal(lv.ghost_gids["lower"].numpy(),
                              down.off + down.send_up_ids.numpy().astype(np.int64))
        assert np.array_equal(lv.ghost_gids["upper"].numpy(),
                              up.off + up.send_down_ids.numpy().astype(np.int64))


@pytest.mark.parametrize("world,counts,p", [(2, (3, 4, 8), 4), (3, (4, 3, 12), 2), (3, (2, 3, 12), 3)])
def test_slab_layout_host(world, counts, p):
    """Host logic of the cfg3 slabs (no GPU): owned slices partition the
    block-major numbering; each rank's element map, pulled back to global ids
    through [owned | bottom ghost | top+1 ghost], is the global map of its
    elements; the exchanged planes are the neighbours' owned planes."""
    import torch
    from paper_1910_03032_b200 import dist_box as D, structured as S
    cpu = torch.device("cpu")
    m = S.box_mesh(counts, perturb=0.0)
    g = S.BoxSpace(m, p, block=2, device=cpu)
    ged = np.asarray(g.element_dofs)
    layers = D.slab_layers(counts[2], world, 4)
    lvs = [D.SlabLevel(m, p, 2, layers, r, world, cpu) for r in range(world)]
    assert [lv.off for lv in lvs] == list(np.cumsum([0] + [lv.n_own for lv in lvs[:-1]]))
    ne_layer = counts[0] * counts[1]

    def plane_ids(gz):
        ids, _ = S.box_lattice_ids(counts, p, 2, cpu, gz_range=(gz, gz + 1))
        return ids.reshape(-1).numpy()

    for r, lv in enumerate(lvs):
        parts = [np.arange(lv.off, lv.off + lv.n_own)]
        if lv.down:
            parts.append(plane_ids(lv.e0 * p))
        if lv.up:
            parts.append(plane_ids(lv.e1 * p + 1))
        l2g = np.concatenate(parts)
        assert l2g.shape[0] == lv.n_local
        e0, e1 = layers[r]
        assert np.array_equal(l2g[np.asarray(lv.element_dofs)], ged[e0 * ne_layer:e1 * ne_layer])
        if lv.down:  # bottom ghost <- rank-1's owned top plane
            dn = lvs[r - 1]
            assert np.array_equal(plane_ids(lv.e0 * p), dn.off + dn.top_plane.numpy())
        if lv.up:  # top+1 ghost <- rank+1's owned bottom+1 plane
            upl = lvs[r + 1]
            assert np.array_equal(plane_ids(lv.e1 * p + 1), upl.off + upl.bot_plus1.numpy())


@pytest.mark.gpu
def test_sharded_cfg3_default_hierarchy_matches_single_gpu():
    """cfg3 shape at 2.1M DoFs with the default hierarchy (Q1 level above
    max_coarse: sharded Q1, agglomerated h-coarse levels) on 1, 2 and 4
    ranks: equal iteration counts, solutions equal to rounding."""
    from paper_1910_03032_b200 import dist_box as D, solvers, structured as S
    counts, p = (32, 32, 32), 4
    cfg = solvers.SolverConfig(rel_tol=1e-8, max_iters=300)
    mesh = S.box_mesh(counts, perturb=0.05, seed=1)
    ref = S.helmholtz_box_problem(counts, p, c=10.0)
    x_ref, rep_ref = solvers.cg(ref["A"], ref["b"], precond=ref["M"], config=cfg)
    x_ref = x_ref.cpu().numpy()
    for world in (2, 4):
        def fn(comm):
            pr = D.helmholtz_slab_problem(comm, counts, p, c=10.0, mesh=mesh)
            lv = pr["level"]
            x, rep = D.dist_cg(pr["A"], pr["b"], pr["M"], comm, lv.n_own, cfg)
            return x[:lv.n_own].cpu().numpy(), rep.iterations, pr["M"].q1_sharded
        out = D.run_threads(world, fn)
        assert all(o[2] for o in out)
        assert all(o[1] == rep_ref.iterations for o in out), ([o[1] for o in out], rep_ref.iterations)
        assert rel_err(np.concatenate([o[0] for o in out]), x_ref) < 1e-12
