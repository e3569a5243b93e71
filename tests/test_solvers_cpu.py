"""CPU: LOR setup, the C++ ILU(0) factorisation and the solver oracle against
the reference's golden fixtures (solvers.npz)."""

import numpy as np
import pytest

from oracle import krylov, sumfact
from paper_1910_03032_b200 import lor, vec
from tests.cases import build, load, manifest, rel_err

SOLVE = {c["name"]: c for c in manifest()["solvers"]}


@pytest.fixture(scope="module")
def gold():
    return load("solvers")


def test_ilu0_host_factor_matches_reference_numba(gold):
    data = gold["ilu/data_in"].astype(np.float64).copy()
    fail = vec.ilu0_factor_host(gold["ilu/indptr"], gold["ilu/indices"], data)
    assert fail == int(gold["ilu/fail"][0]) == -1
    ref = gold["ilu/data_out"]
    assert np.max(np.abs(data - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_ilu0_oracle_matches_host_factor(gold):
    ip, ix = gold["ilu/indptr"], gold["ilu/indices"]
    a = gold["ilu/data_in"].astype(np.float64).copy()
    b = a.copy()
    assert krylov.ilu0(ip, ix, a) == vec.ilu0_factor_host(ip, ix, b) == -1
    assert np.max(np.abs(a - b)) <= 1e-13 * np.max(np.abs(b))


def test_ilu0_zero_pivot_reports_row():
    # 2x2 with a zero pivot in row 0
    ip = np.array([0, 2, 4])
    ix = np.array([0, 1, 0, 1])
    d = np.array([0.0, 1.0, 1.0, 1.0])
    assert vec.ilu0_factor_host(ip, ix, d) == 0


def test_first_touch_ordering_is_a_permutation():
    _, sp_, _ = build(3, (3, 2, 2), None, 0.0, 3)
    order = lor.first_touch_ordering(sp_)
    assert np.array_equal(np.sort(order), np.arange(sp_.ndofs_scalar))
    assert order[0] == sp_.element_dofs[0, 0]


@pytest.mark.parametrize("name", ["cfg1_poisson", "3d_p4_helmholtz", "2d_p7_helmholtz_pert"])
def test_lor_levels_and_oracle_vcycle(name, gold):
    from paper_1910_03032_b200 import spaces
    c = SOLVE[name]
    m, sp_, geom = build(c["d"], c["counts"], None, c["perturb"], c["p"])
    mats, spaces_, transfers = [], [], []
    for deg in lor.degree_ladder(c["p"]):
        lsp = sp_ if deg == c["p"] else spaces.FESpace(m, deg)
        mats.append(lor.lor_matrix(lsp, c["kind"], nu=1.0, c=c["c"],
                                   constrained=lsp.boundary_dof_set()))
        if spaces_:
            transfers.append(lor.nodal_interpolation(spaces_[-1], lsp))
        spaces_.append(lsp)
    assert [A.nnz for A in mats] == list(gold[name + "/lor_nnz"])
    vc = krylov.VCycle(mats, transfers, [lor.first_touch_ordering(s) for s in spaces_[:-1]])
    r = np.random.default_rng(99).standard_normal(sp_.ndofs)
    assert rel_err(vc(r), gold[name + "/vcycle"]) < 1e-10


def test_oracle_cg_iterations_cfg1(gold):
    from paper_1910_03032_b200 import spaces
    c = SOLVE["cfg1_poisson"]
    m, sp_, geom = build(c["d"], c["counts"], None, c["perturb"], c["p"])
    op = sumfact.make_square("stiffness", sp_, geom)
    bdr = sp_.boundary_dof_set()
    mats, ss, tr = [], [], []
    for deg in lor.degree_ladder(4):
        lsp = sp_ if deg == 4 else spaces.FESpace(m, deg)
        mats.append(lor.lor_matrix(lsp, "stiffness", constrained=lsp.boundary_dof_set()))
        if ss:
            tr.append(lor.nodal_interpolation(ss[-1], lsp))
        ss.append(lsp)
    vc = krylov.VCycle(mats, tr, [lor.first_touch_ordering(s) for s in ss[:-1]])
    A = lambda v: sumfact.constrained_apply(op, bdr, v)  # noqa: E731
    b = np.random.default_rng(0).standard_normal(sp_.ndofs)
    b[bdr] = 0.0
    x, its, _ = krylov.cg(A, b, precond=vc, rel_tol=1e-8, max_iters=300)
    assert abs(its - c["iterations"][0]) <= 1
    assert rel_err(x, gold["cfg1_poisson/x0"]) < 1e-6


def test_gc_pause_nests_across_threads():
    """The CG-graph capture pauses cyclic GC; in-process ranks capture
    concurrently, so the pause is reference counted and restores the
    caller's setting only when the last capture ends."""
    import gc
    import threading
    from paper_1910_03032_b200 import solvers as S
    assert gc.isenabled()
    barrier = threading.Barrier(3)
    seen = []

    def rank():
        S._gc_pause(True)
        barrier.wait()
        seen.append(gc.isenabled())
        barrier.wait()
        S._gc_pause(False)

    ts = [threading.Thread(target=rank) for _ in range(2)]
    for t in ts:
        t.start()
    barrier.wait()
    barrier.wait()
    for t in ts:
        t.join()
    assert seen == [False, False]
    assert gc.isenabled()
    gc.disable()
    try:
        S._gc_pause(True)
        S._gc_pause(False)
        assert not gc.isenabled()  # a caller that had GC off keeps it off
    finally:
        gc.enable()
