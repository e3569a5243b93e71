"""Projection stepping (cfg5 caller, timeint.py:218-388): BDF/EXT weights on
CPU; the device stepper against the reference's periodic 3D Taylor-Green run
(extras.npz, tests/golden/make_golden.py) on the GPU."""

import numpy as np
import pytest

from tests.cases import load, manifest, rel_err


def test_bdf_coefficients_match_reference_tables():
    from paper_1910_03032_b200 import timeint
    for k, b, a in [(1, (1.0, -1.0), (1.0,)), (2, (1.5, -2.0, 0.5), (2.0, -1.0)),
                    (3, (11.0 / 6.0, -3.0, 1.5, -1.0 / 3.0), (3.0, -3.0, 1.0))]:
        s = timeint.bdf_coefficients(k)
        assert np.array_equal(s.b, np.array(b)) and np.array_equal(s.a, np.array(a))
    with pytest.raises(ValueError):
        timeint.bdf_coefficients(4)


@pytest.mark.gpu
def test_projection_stepper_taylor_green_matches_reference():
    from paper_1910_03032_b200 import geometry, spaces, timeint
    c = manifest()["projection"][0]
    gold = load("extras")
    m = geometry.cartesian_mesh(tuple(c["counts"]), lows=(-np.pi,) * 3, highs=(np.pi,) * 3,
                                periodic=(True,) * 3)
    vs = spaces.FESpace(m, c["p"], vdim=3)
    ps = spaces.FESpace(m, c["p"])
    geom = geometry.compute_geometric_factors(m, vs.basis.quad)
    st = timeint.ProjectionStepper(vs, ps, geom, k=c["k"], dt=c["dt"], nu=c["nu"],
                                   smoother="global")
    st.initialize(gold["tgv3d_p3/u0"])
    for want in c["iterations"]:
        r = st.step()
        got = [r.mass_iters, r.pressure_iters, r.helmholtz_iters]
        assert all(abs(g - w) <= 1 for g, w in zip(got, want)), (got, want)
    u = st.u.cpu().numpy()
    p = st.p.cpu().numpy()
    assert rel_err(u, gold["tgv3d_p3/u"]) < 1e-8
    assert rel_err(p, gold["tgv3d_p3/p"]) < 1e-6
    assert st.kinetic_energy() == pytest.approx(float(gold["tgv3d_p3/energy"][0]), rel=1e-10)


@pytest.mark.gpu
def test_box_projection_stepper_taylor_green_matches_reference():
    """Scale-mode projection stepper (periodic BoxSpace numbering, device-built
    pure-Neumann / Helmholtz block-ILU hierarchies) on the reference's 3D
    periodic Taylor-Green golden.  Its preconditioners are the block-Jacobi
    ILU(0) ones, so its iteration counts are pinned to the parity stepper
    with the same smoother (+-1) and its fields / energy to the reference's
    golden after four BDF3 steps."""
    from paper_1910_03032_b200 import geometry, spaces, structured as S, timeint
    c = manifest()["projection"][0]
    gold = load("extras")
    m = geometry.cartesian_mesh(tuple(c["counts"]), lows=(-np.pi,) * 3, highs=(np.pi,) * 3,
                                periodic=(True,) * 3)
    vs = spaces.FESpace(m, c["p"], vdim=3)
    ps = spaces.FESpace(m, c["p"])
    geom = geometry.compute_geometric_factors(m, vs.basis.quad)
    par = timeint.ProjectionStepper(vs, ps, geom, k=c["k"], dt=c["dt"], nu=c["nu"],
                                    smoother="block")
    par.initialize(gold["tgv3d_p3/u0"])
    counts, per = tuple(c["counts"]), (True, True, True)
    ids, _ = S.box_lattice_ids(counts, c["p"], 2, periodic=per)
    perm = np.full(ps.ndofs_scalar, -1, dtype=np.int64)
    perm[ps.element_dofs.ravel()] = S.lattice_element_dofs(ids, c["p"], per).numpy().ravel()
    ns = ps.ndofs_scalar
    vperm = np.concatenate([perm + k * ns for k in range(3)])
    st = timeint.BoxProjectionStepper(m, c["p"], k=c["k"], dt=c["dt"], nu=c["nu"])
    u0 = np.empty(3 * ns)
    u0[vperm] = gold["tgv3d_p3/u0"]
    st.initialize(u0)
    for _ in range(c["steps"]):
        r, rp = st.step(), par.step()
        got = [r.mass_iters, r.pressure_iters, r.helmholtz_iters]
        want = [rp.mass_iters, rp.pressure_iters, rp.helmholtz_iters]
        assert all(abs(g - w) <= 1 for g, w in zip(got, want)), (got, want)
    u = st.u.cpu().numpy()[vperm]
    p = st.p.cpu().numpy()[perm]
    assert rel_err(u, par.u.cpu().numpy()) < 1e-8
    assert rel_err(u, gold["tgv3d_p3/u"]) < 1e-7
    assert rel_err(p, gold["tgv3d_p3/p"]) < 1e-5
    assert st.kinetic_energy() == pytest.approx(float(gold["tgv3d_p3/energy"][0]), rel=1e-9)
    assert isinstance(st.pressure_pre, S.BoxLORPreconditioner)
