"""CPU: the product's setup code (mesh, numbering, geometry) reproduces the
reference bit for bit on the golden meshes (fespace.py:71-217,
mesh.py:63-267)."""

import numpy as np
import pytest

from paper_1910_03032_b200 import geometry, quadrature, spaces
from tests.cases import load, manifest

NUM = manifest()["numbering"]


@pytest.fixture(scope="module")
def gold():
    return load("numbering")


@pytest.mark.parametrize("case", NUM, ids=[c["key"] for c in NUM])
def test_numbering_and_geometry(case, gold):
    k = case["key"]
    per = tuple(case["periodic"]) if case["periodic"] else None
    m = geometry.perturb_mesh(geometry.cartesian_mesh(tuple(case["counts"]), periodic=per), 0.08,
                              seed=11)
    sp = spaces.FESpace(m, case["p"])
    assert sp.ndofs_scalar == case["ndofs"]
    assert np.array_equal(sp.element_dofs, gold[k + "/element_dofs"])
    assert np.array_equal(sp.boundary_dof_set(), gold[k + "/boundary"])
    assert np.array_equal(sp.dof_owner_elem, gold[k + "/owner_elem"])
    assert np.array_equal(m.corners, gold[k + "/corners"])
    g = geometry.compute_geometric_factors(m, sp.basis.quad)
    assert np.allclose(g.detj, gold[k + "/detj"], rtol=1e-14, atol=0)
    assert np.allclose(g.jinv, gold[k + "/jinv"], rtol=1e-13, atol=1e-14)


def test_basis_matrices_reproduce_polynomials():
    for p in range(1, 12):
        b = quadrature.make_basis(p)
        x = b.quad.points
        # B interpolates x^p exactly, D differentiates it
        vals = b.nodes ** p
        assert np.allclose(b.B @ vals, x ** p, atol=1e-12)
        assert np.allclose(b.D @ vals, p * x ** (p - 1), atol=1e-10)
        Dq = quadrature.differentiation_matrix(x)
        assert np.allclose(Dq @ b.B, b.D, atol=1e-11)


def test_number_dofs_rejects_bad_dim():
    m = geometry.cartesian_mesh((2, 2))
    m.dim = 4
    with pytest.raises(ValueError):
        spaces.number_dofs(m, 2)


def test_large_structured_numbering_is_fast():
    import time
    m = geometry.cartesian_mesh((20, 20, 20))
    t = time.perf_counter()
    sp = spaces.FESpace(m, 4)
    assert time.perf_counter() - t < 20
    assert sp.ndofs_scalar == 81 ** 3
