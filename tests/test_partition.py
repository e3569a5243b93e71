"""CPU: slab partition + cut-plane halo sum + distributed dot, world_size 2 and
3 over gloo (the multi-GPU path's host logic).  The local apply
here is the numpy oracle, so the test exercises exactly the partition and
communication code that runs unchanged over NCCL on GPUs."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class _OracleLocalOp:
    """Local (slab) operator from the oracle, with the device-op interface."""

    def __init__(self, kind, lsp, geom_full, part, c, nu):
        from oracle import sumfact
        B, D = lsp.basis.eval_matrices_at(geom_full.rule.points)
        lo, hi = part.e_lo, part.e_hi
        wdet = c * sumfact.mass_factor(geom_full.detj[lo:hi], geom_full.w)
        stiff = sumfact.stiffness_factor(geom_full.detj[lo:hi], geom_full.jinv[lo:hi],
                                         geom_full.w, nu)
        self.space = lsp
        self.shape = (lsp.ndofs, lsp.ndofs)
        self._f = lambda x: sumfact.square_apply(kind, lsp.element_dofs, lsp.ndofs_scalar,
                                                 lsp.vdim, B, D, lsp.dim, x, wdet, stiff)

    def apply_into(self, x, y, stream=None):
        y.copy_(torch.from_numpy(self._f(x.numpy())))
        return y


def _worker(rank, world, port, d, counts, p, vdim, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sumfact
        from paper_1910_03032_b200 import geometry, partition, spaces
        m = geometry.perturb_mesh(geometry.cartesian_mesh(counts), 0.05, seed=2)
        sp = spaces.FESpace(m, p, vdim=vdim)
        geom = geometry.compute_geometric_factors(m, sp.basis.quad)
        part = partition.SlabPartition(sp, rank, world)
        lsp = part.local_space()
        op = partition.DistributedOperator(_OracleLocalOp("helmholtz", lsp, geom, part, 3.0, 0.7),
                                           part)
        x = np.random.default_rng(0).standard_normal(sp.ndofs)
        ns = sp.ndofs_scalar
        xl = np.concatenate([part.scatter_global(x[c * ns:(c + 1) * ns]) for c in range(vdim)])
        yl = torch.empty(xl.size, dtype=torch.float64)
        op.apply_into(torch.from_numpy(xl), yl)
        y_ref = sumfact.make_square("helmholtz", sp, geom, c=3.0, nu=0.7)(x)
        nl = part.n_local
        err = 0.0
        for c in range(vdim):
            ref = y_ref[c * ns:(c + 1) * ns][part.global_ids]
            got = yl[c * nl:(c + 1) * nl].numpy()
            err = max(err, np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
        xs = torch.from_numpy(xl[:nl])
        gdot = partition.distributed_dot(xs, xs, part).item()
        ref_dot = float(x[:ns] @ x[:ns])
        q.put((rank, err, abs(gdot - ref_dot) / ref_dot, part.n_owned))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,d,counts,p,vdim", [
    (2, 3, (3, 2, 4), 3, 1),
    (3, 3, (2, 3, 5), 2, 1),
    (2, 2, (4, 5), 4, 2),
])
def test_slab_halo_apply_and_dot(world, d, counts, p, vdim):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, counts, p, vdim, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    from paper_1910_03032_b200 import geometry, spaces
    n_total = spaces.FESpace(geometry.cartesian_mesh(counts), p).ndofs_scalar
    assert sum(r[3] for r in res) == n_total  # owned sets partition the DoFs
    for rank, err, derr, _ in res:
        assert err < 1e-13, (rank, err)
        assert derr < 1e-13, (rank, derr)


def test_partition_bookkeeping():
    from paper_1910_03032_b200 import geometry, partition, spaces
    m = geometry.cartesian_mesh((3, 3, 6))
    sp = spaces.FESpace(m, 2)
    parts = [partition.SlabPartition(sp, r, 3) for r in range(3)]
    owned = np.concatenate([pt.global_ids[:pt.n_owned] for pt in parts])
    assert np.array_equal(np.sort(owned), np.arange(sp.ndofs_scalar))
    # neighbours agree on the shared cut-plane DoFs
    for r in range(2):
        a = parts[r].global_ids[parts[r].shared[r + 1]]
        b = parts[r + 1].global_ids[parts[r + 1].shared[r]]
        assert np.array_equal(a, b) and a.size == (2 * 3 + 1) ** 2
    with pytest.raises(ValueError):
        partition.SlabPartition(sp, 0, 7)


def _slab_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sumfact
        from paper_1910_03032_b200 import geometry, partition
        slab = partition.StructuredSlab((3, 2), 2, 3, rank, world, perturb=0.05)
        geom = geometry.compute_geometric_factors(slab.mesh, slab.space.basis.quad)
        f = sumfact.make_square("stiffness", slab.space, geom)
        halo = partition.HaloExchange(slab)
        y = torch.from_numpy(f(np.ones(slab.n_local)))
        halo.sum(y)
        # stiffness kills constants globally only after the halo sum
        q.put((rank, float(y.abs().max()), int(slab.owned_mask.sum())))
    finally:
        dist.destroy_process_group()


def test_structured_slab_halo_kills_constants():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    from paper_1910_03032_b200 import geometry, spaces
    n_total = spaces.FESpace(geometry.cartesian_mesh((3, 2, 6)), 3).ndofs_scalar
    assert sum(r[2] for r in res) == n_total
    for rank, err, _ in res:
        assert err < 1e-12, (rank, err)
