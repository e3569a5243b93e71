"""Boundary surface functionals of the bounded-domain projection step
(mfop.py:623-807) against the reference's own outputs (boundary.npz,
tests/golden/make_golden.py): the setup-built face matrices on CPU, the
device SpMV and the bounded ProjectionStepper on the GPU."""

import numpy as np
import pytest

from tests.cases import load, manifest, rel_err


def _case(c):
    from paper_1910_03032_b200 import geometry, spaces
    m = geometry.perturb_mesh(geometry.cartesian_mesh(tuple(c["counts"])), c["perturb"], seed=11)
    vs = spaces.FESpace(m, c["p_v"], vdim=c["d"])
    ps = spaces.FESpace(m, c["p_p"])
    u = np.random.default_rng(c["seed"]).standard_normal(vs.ndofs)
    return m, vs, ps, u


def _flux_field(x):
    from tests.golden.make_golden import flux_field
    return flux_field(x)


@pytest.mark.parametrize("c", manifest()["boundary"], ids=lambda c: c["name"])
def test_face_matrices_match_reference(c):
    from paper_1910_03032_b200 import boundary
    gold = load("boundary")
    _, vs, ps, u = _case(c)
    R = boundary.RotationalMatrix(vs, ps, nu=c["nu"], attributes=c["attributes"],
                                  n_quad=c["n_quad"])
    want = gold[c["name"] + "/rot"]
    assert rel_err(R.matrix @ u, want) < 1e-12
    assert abs(np.sum(R.matrix @ u)) < 1e-10 * np.linalg.norm(want)  # orthogonal to constants
    N = boundary.NormalFluxMatrix(ps, attributes=c["attributes"], n_quad=c["n_quad"])
    g = _flux_field(N.points)
    assert rel_err(N.matrix @ g.reshape(-1), gold[c["name"] + "/flux"]) < 1e-12


def test_face_matrix_shapes_and_errors():
    from paper_1910_03032_b200 import boundary, geometry, spaces
    m = geometry.cartesian_mesh((2, 2))
    vs = spaces.FESpace(m, 2, vdim=2)
    ps = spaces.FESpace(m, 2)
    with pytest.raises(ValueError):
        boundary.RotationalMatrix(ps, ps)
    R = boundary.RotationalMatrix(vs, ps)
    assert R.matrix.shape == (ps.ndofs, vs.ndofs)
    N = boundary.NormalFluxMatrix(ps)
    assert N.points.shape == (8 * 4, 2)  # 8 boundary faces x (p+2) points


@pytest.mark.gpu
@pytest.mark.parametrize("c", manifest()["boundary"], ids=lambda c: c["name"])
def test_boundary_functionals_on_device(c):
    import torch

    from paper_1910_03032_b200 import boundary, device as dev
    boundary.clear_cache()
    gold = load("boundary")
    _, vs, ps, u = _case(c)
    r = boundary.boundary_rotational_rhs(vs, ps, dev.to_device(u), nu=c["nu"],
                                         attributes=c["attributes"], n_quad=c["n_quad"])
    assert isinstance(r, torch.Tensor) and r.is_cuda
    assert rel_err(r.cpu().numpy(), gold[c["name"] + "/rot"]) < 1e-12
    f = boundary.boundary_normal_flux(ps, _flux_field, attributes=c["attributes"],
                                      n_quad=c["n_quad"])
    assert rel_err(f, gold[c["name"] + "/flux"]) < 1e-12


@pytest.mark.gpu
def test_bounded_projection_stepper_matches_reference():
    from paper_1910_03032_b200 import geometry, spaces, timeint
    from tests.golden.make_golden import tgv2d_exact
    c = manifest()["projection_bounded"][0]
    gold = load("boundary")
    m = geometry.perturb_mesh(geometry.cartesian_mesh(tuple(c["counts"]), lows=(-1.0, -1.0),
                                                      highs=(1.0, 1.0)), c["perturb"], seed=11)
    vs = spaces.FESpace(m, c["p"], vdim=2)
    ps = spaces.FESpace(m, c["p"])
    geom = geometry.compute_geometric_factors(m, vs.basis.quad)
    st = timeint.ProjectionStepper(vs, ps, geom, k=c["k"], dt=c["dt"], nu=c["nu"],
                                   dirichlet=tgv2d_exact(c["nu"]), smoother="global")
    st.initialize(gold["tgv2d_box_p4/u0"])
    for want in c["iterations"]:
        r = st.step()
        got = [r.mass_iters, r.pressure_iters, r.helmholtz_iters]
        assert all(abs(g - w) <= 1 for g, w in zip(got, want)), (got, want)
    assert rel_err(st.u.cpu().numpy(), gold["tgv2d_box_p4/u"]) < 1e-8
    assert rel_err(st.p.cpu().numpy(), gold["tgv2d_box_p4/p"]) < 1e-6
