"""GPU: Stokes block operator, block-triangular preconditioner and the FGMRES
lid-cavity solves (cfg4 caller) against the reference's goldens (stokes.npz)."""

import numpy as np
import pytest

from tests.cases import load, manifest, rel_err

pytestmark = pytest.mark.gpu

CASES = {c["name"]: c for c in manifest()["stokes"]}


def lid(X):
    out = np.zeros_like(X)
    out[np.abs(X[:, 1] - 1.0) < 1e-12, 0] = 1.0
    return out


@pytest.fixture(scope="module")
def gold():
    return load("stokes")


@pytest.mark.parametrize("smoother", ["global", "block"])
@pytest.mark.parametrize("name", sorted(CASES))
def test_lid_cavity_matches_reference(name, smoother, gold, monkeypatch):
    from paper_1910_03032_b200 import geometry, solvers, spaces, stokes
    monkeypatch.setattr(solvers, "DEFAULT_SMOOTHER", smoother)
    c = CASES[name]
    m = geometry.cartesian_mesh(tuple(c["counts"]))
    vs = spaces.FESpace(m, c["p"], vdim=c["d"])
    ps = spaces.FESpace(m, c["p"] - 1)
    geom = geometry.compute_geometric_factors(m, vs.basis.quad)
    S = stokes.StokesSystem(vs, ps, geom, nu=1.0, alpha_dt=c["alpha_dt"])
    x = np.random.default_rng(3).standard_normal(S.K.shape[0])
    assert rel_err(S.K.apply(x), gold[name + "/Kx"]) < 1e-12
    if smoother == "global":  # the reference's cycle, reproduced to rounding
        assert rel_err(S.P.apply(x), gold[name + "/Px"]) < 1e-9
    u, p, rep = S.solve(g=lid, config=solvers.SolverConfig(rel_tol=1e-8, max_iters=200))
    assert rep.converged
    assert abs(rep.iterations - c["iterations"]) <= 1, (rep.iterations, c["iterations"])
    assert rel_err(u, gold[name + "/u"]) < 1e-6
    assert rel_err(p, gold[name + "/p"]) < 1e-5


def test_block_operator_rejects_bad_shape():
    from paper_1910_03032_b200 import geometry, spaces, stokes
    m = geometry.cartesian_mesh((3, 3))
    vs = spaces.FESpace(m, 2, vdim=2)
    ps = spaces.FESpace(m, 1)
    geom = geometry.compute_geometric_factors(m, vs.basis.quad)
    S = stokes.StokesSystem(vs, ps, geom)
    with pytest.raises(ValueError, match="shape"):
        S.K.apply(np.zeros(S.K.shape[0] + 1))
    with pytest.raises(ValueError):
        stokes.StokesSystem(vs, spaces.FESpace(m, 2), geom)


@pytest.mark.parametrize("name", ["cav2d_p2", "cav2d_p4", "cav3d_p2"])
def test_minres_lid_cavity_matches_reference_solution(name, gold):
    """Block-diagonal-preconditioned MINRES on the symmetric saddle form
    (north star's Stokes solver; no reference counterpart) reaches the
    reference's FGMRES solution of the same cavity."""
    from paper_1910_03032_b200 import geometry, solvers, spaces, stokes
    c = CASES[name]
    m = geometry.cartesian_mesh(tuple(c["counts"]))
    vs = spaces.FESpace(m, c["p"], vdim=c["d"])
    ps = spaces.FESpace(m, c["p"] - 1)
    geom = geometry.compute_geometric_factors(m, vs.basis.quad)
    S = stokes.StokesSystem(vs, ps, geom, nu=1.0)
    u, p, rep = S.solve_minres(g=lid, config=solvers.SolverConfig(rel_tol=1e-12, max_iters=2000))
    assert rep.converged, rep
    assert rel_err(u, gold[name + "/u"]) < 1e-6
    assert rel_err(p, gold[name + "/p"]) < 1e-5
