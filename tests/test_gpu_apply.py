"""GPU parity: the CUDA operator path vs the reference golden vectors and the
oracle (1e-12 relative, the north-star bar), determinism, and properties at
full benchmark sizes."""

import numpy as np
import pytest

from oracle import sumfact
from tests.cases import build, load, manifest, rel_err

pytestmark = pytest.mark.gpu

MAN = manifest()
APPLY = {c["name"]: c for c in MAN["apply"]}
MIXED = {c["name"]: c for c in MAN["mixed"]}
TOL = 1e-12


@pytest.fixture(scope="module")
def gold():
    return load("apply")


def _make(c, sp, geom):
    from paper_1910_03032_b200 import mfop
    kw = {"mass": {}, "stiffness": {"nu": c["nu"]}, "helmholtz": {"c": c["c"], "nu": c["nu"]}}
    return mfop.setup(c["kind"], space=sp, geom=geom, **kw[c["kind"]])


@pytest.mark.parametrize("name", sorted(APPLY))
def test_square_apply_matches_reference(name, gold):
    from paper_1910_03032_b200 import geometry, mfop
    c = APPLY[name]
    m, sp, geom = build(c["d"], c["counts"], c["periodic"], c["perturb"], c["p"], c["vdim"])
    x = np.random.default_rng(c["seed"]).standard_normal(sp.ndofs)
    op = _make(c, sp, geom)
    y = op.apply(x)
    assert isinstance(y, np.ndarray) and y.shape == x.shape
    assert rel_err(y, gold[name + "/y"]) < TOL
    # same operator with factors built on the device from the corners
    op_dev = _make(c, sp, geometry.DeviceGeometry(m, sp.basis.quad))
    assert rel_err(op_dev.apply(x), gold[name + "/y"]) < TOL
    if c["d"] == 3 and c["p"] <= 8:
        assert op.fast_path, "3D n_q = p+2 must run the fused sm_100a kernel"
    if name + "/yc" in gold.files:
        bd = sp.expand_dofs(sp.boundary_dof_set())
        yc = mfop.ConstrainedOperator(op, bd).apply(x)
        assert rel_err(yc, gold[name + "/yc"]) < TOL


@pytest.mark.parametrize("name", sorted(MIXED))
def test_mixed_apply_matches_reference(name, gold):
    from paper_1910_03032_b200 import geometry, mfop, spaces
    c = MIXED[name]
    m, vs, geom = build(c["d"], c["counts"], c["periodic"], c["perturb"], c["pv"], vdim=c["d"])
    ps = spaces.FESpace(m, c["pp"])
    rng = np.random.default_rng(c["seed"])
    q = rng.standard_normal(ps.ndofs_scalar)
    v = rng.standard_normal(vs.ndofs)
    for g in (geom, geometry.DeviceGeometry(m, vs.basis.quad)):
        G = mfop.GradientOperator(vs, ps, g)
        D = mfop.DivergenceOperator(vs, ps, g)
        assert rel_err(G.apply(q), gold[name + "/G"]) < TOL
        assert rel_err(G.apply_transpose(v), gold[name + "/Gt"]) < TOL
        assert rel_err(D.apply(v), gold[name + "/D"]) < TOL


def test_torch_operands_stay_on_device():
    import torch
    from paper_1910_03032_b200 import mfop
    _, sp, geom = build(3, (3, 2, 2), None, 0.05, 4)
    op = mfop.HelmholtzOperator(sp, geom, 10.0)
    x = np.random.default_rng(0).standard_normal(sp.ndofs)
    yd = op.apply(torch.from_numpy(x).cuda())
    assert yd.is_cuda and yd.dtype == torch.float64
    assert np.array_equal(yd.cpu().numpy(), op.apply(x))
    with pytest.raises(ValueError, match="shape"):
        op.apply(np.zeros(sp.ndofs + 1))


def test_apply_is_deterministic_and_matches_oracle():
    from paper_1910_03032_b200 import mfop
    for p in (2, 5, 8):
        _, sp, geom = build(3, (4, 3, 3), None, 0.05, p)
        op = mfop.HelmholtzOperator(sp, geom, 10.0)
        ref = sumfact.make_square("helmholtz", sp, geom, c=10.0)
        x = np.random.default_rng(p).standard_normal(sp.ndofs)
        y1 = op.apply(x)
        y2 = op.apply(x)
        assert np.array_equal(y1, y2)
        assert rel_err(y1, ref(x)) < TOL


def test_restriction_scatter_is_bitwise_bincount():
    from paper_1910_03032_b200 import mfop
    _, sp, _ = build(3, (3, 3, 2), None, 0.05, 3)
    r = mfop.restriction(sp)
    loc = np.random.default_rng(1).standard_normal(sp.element_dofs.shape)
    assert np.array_equal(r.scatter_add(loc), sumfact.scatter_add(sp.element_dofs, loc,
                                                                  sp.ndofs_scalar))
    x = np.random.default_rng(2).standard_normal(sp.ndofs_scalar)
    assert np.array_equal(r.gather(x), x[sp.element_dofs])


def test_interior_split_matches_full_scatter():
    """The fused kernel writes element-interior DoFs directly and sums shared
    ones through the transposed map; the total equals the E-vector path."""
    from paper_1910_03032_b200 import mfop
    _, sp, geom = build(3, (3, 2, 2), None, 0.05, 4)
    x = np.random.default_rng(3).standard_normal(sp.ndofs)
    fast = mfop.StiffnessOperator(sp, geom)
    assert fast.fast_path
    ref = sumfact.make_square("stiffness", sp, geom)
    assert rel_err(fast.apply(x), ref(x)) < TOL


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_full_size_properties(p):
    """cfg2-sized meshes (~2M DoFs here): symmetry, constants in the kernel
    of the stiffness, mass of ones = volume, Helmholtz = c M + L."""
    import torch
    from paper_1910_03032_b200 import geometry, mfop, spaces
    n = max(2, round((2.0e6) ** (1 / 3) / p))
    m = geometry.perturb_mesh(geometry.cartesian_mesh((n, n, n)), 0.05, seed=1)
    sp = spaces.FESpace(m, p)
    g = geometry.DeviceGeometry(m, sp.basis.quad)
    H = mfop.HelmholtzOperator(sp, g, 10.0)
    M = mfop.MassOperator(sp, g)
    L = mfop.StiffnessOperator(sp, g)
    gen = torch.Generator(device="cuda").manual_seed(p)
    x = torch.randn(sp.ndofs, dtype=torch.float64, device="cuda", generator=gen)
    z = torch.randn(sp.ndofs, dtype=torch.float64, device="cuda", generator=gen)
    hx = H.apply(x)
    lin = 10.0 * M.apply(x) + L.apply(x)
    assert (torch.linalg.norm(hx - lin) / torch.linalg.norm(hx)).item() < 1e-13
    sym = (z @ hx - x @ H.apply(z)).abs().item() / (torch.linalg.norm(z) *
                                                   torch.linalg.norm(hx)).item()
    assert sym < 1e-13
    ones = torch.ones(sp.ndofs, dtype=torch.float64, device="cuda")
    assert abs((ones @ M.apply(ones)).item() - 1.0) < 1e-12
    assert L.apply(ones).abs().max().item() < 1e-10


CONV = {c["name"]: c for c in MAN.get("convection", [])}


@pytest.mark.parametrize("device_geom", [False, True])
@pytest.mark.parametrize("name", sorted(CONV))
def test_convection_matches_reference(name, device_geom):
    """ConvectionOperator on the device vs the reference's (extras.npz)."""
    from paper_1910_03032_b200 import geometry, mfop
    c = CONV[name]
    gold = load("extras")
    m, vs, geom = build(c["d"], c["counts"], c["periodic"], c["perturb"], c["p"], vdim=c["d"])
    if device_geom:
        geom = geometry.DeviceGeometry(m, vs.basis.quad)
    op = mfop.setup("convection", vspace=vs, geom=geom)
    u = np.random.default_rng(c["seed"]).standard_normal(vs.ndofs)
    assert rel_err(op.apply(u), gold[name + "/y"]) < 1e-12


def test_restriction_with_untouched_dofs_is_bincount():
    """DoFs no element touches (the ghost planes of a slab-local space) sum
    to zero in the class-major E->L layout -- bitwise np.bincount."""
    from paper_1910_03032_b200 import geometry, mfop, spaces

    class Padded:
        def __init__(self, sp, extra):
            self.dim, self.p = sp.dim, sp.p
            self.element_dofs = sp.element_dofs
            self.ndofs_scalar = sp.ndofs_scalar + extra

    m = geometry.cartesian_mesh((3, 2, 2))
    for p in (1, 3):
        sp = Padded(spaces.FESpace(m, p), 37)
        r = mfop.Restriction(sp)
        xe = np.random.default_rng(p).standard_normal(sp.element_dofs.shape)
        want = np.bincount(sp.element_dofs.ravel(), weights=xe.ravel(), minlength=sp.ndofs_scalar)
        got = r.scatter_add(xe)
        assert np.array_equal(got, want)


CURL = {c["name"]: c for c in MAN.get("curlcurl", [])}


@pytest.mark.parametrize("device_geom", [False, True])
@pytest.mark.parametrize("name", sorted(CURL))
def test_curlcurl_matches_reference(name, device_geom):
    """CurlCurlOperator on the device vs the reference's (extras.npz)."""
    from paper_1910_03032_b200 import geometry, mfop
    c = CURL[name]
    gold = load("extras")
    m, vs, geom = build(c["d"], c["counts"], c["periodic"], c["perturb"], c["p"], vdim=c["d"])
    if device_geom:
        geom = geometry.DeviceGeometry(m, vs.basis.quad)
    op = mfop.setup("curlcurl", vspace=vs, geom=geom, nu=c["nu"])
    u = np.random.default_rng(c["seed"]).standard_normal(vs.ndofs)
    assert rel_err(op.apply(u), gold[name + "/y"]) < 1e-12
