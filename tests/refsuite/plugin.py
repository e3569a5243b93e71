"""pytest plugin: run the REFERENCE's own test modules against this package.

Import substitution ("directly re-usable as drop-in
acceptance"): the reference's setup modules (basis, mesh, fespace, lor,
kernels) and its assembled-matrix oracle (`mfop.assemble`, the dense
quadrature loops written in the test files) stay the reference's; every
hot-path class / function the tests reach through `flowbench.mfop`,
`flowbench.solvers` and `flowbench.stokes` is replaced by this package's
device implementation before the test modules are imported.  The reference
package comes from oracle/_ref (oracle/build_ref.py); the tests from
oracle/_ref/tests.  Used by tests/test_reference_suite.py:

    python -m pytest oracle/_ref/tests/test_mfop.py -p tests.refsuite.plugin
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/fb_ref_numba_cache")
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref", "site"))

import flowbench  # noqa: E402
import flowbench.lor as _rlor  # noqa: E402
import flowbench.mfop as _rmfop  # noqa: E402
import flowbench.solvers as _rsol  # noqa: E402
import flowbench.stokes as _rst  # noqa: E402

from paper_1910_03032_b200 import _lib, lor, mfop, solvers, stokes  # noqa: E402

assert os.path.abspath(flowbench.__file__).startswith(os.path.join(ROOT, "oracle", "_ref"))

# the hot path plus the f4 caller pieces
SUBSTITUTE = {
    _rmfop: (mfop, ["MassOperator", "StiffnessOperator", "HelmholtzOperator", "GradientOperator",
                    "DivergenceOperator", "ConvectionOperator", "CurlCurlOperator",
                    "ConstrainedOperator", "setup", "boundary_rotational_rhs"]),
    _rsol: (solvers, ["SolverConfig", "SolveReport", "cg", "fgmres", "MeanProjector",
                      "deflate_mean", "DiagonalPreconditioner", "collocated_mass_diagonal",
                      "ILU0Smoother", "LORPreconditioner", "BlockDiagonalPreconditioner",
                      "InnerCG", "_first_touch_ordering"]),
    _rst: (stokes, ["BlockSaddleOperator", "SteadySchurInverse", "UnsteadySchurInverse",
                    "BlockTriangularPreconditioner", "StokesSystem"]),
    # LOR matrices / transfers the V-cycle applies (lor.py:61-131); the
    # refined-mesh builder, Matrix Market export and spectral report stay
    _rlor: (lor, ["lor_matrix", "constrain_matrix", "nodal_interpolation",
                  "coarse_q1_interpolation"]),
}
for _ref_mod, (_ours, _names) in SUBSTITUTE.items():
    for _n in _names:
        setattr(_ref_mod, _n, getattr(_ours, _n))

_launches0 = _lib.lib.fb_launch_count()


def pytest_report_header(config):
    n = sum(len(v[1]) for v in SUBSTITUTE.values())
    return [f"refsuite: reference flowbench from {os.path.dirname(flowbench.__file__)}; "
            f"{n} hot-path names substituted by paper_1910_03032_b200"]


def pytest_sessionfinish(session, exitstatus):
    n = _lib.lib.fb_launch_count() - _launches0
    print(f"\nrefsuite: libfbb200 kernel launches during the run: {n}")
    if n <= 0 and exitstatus == 0:
        session.exitstatus = 3  # nothing ran on the device: the substitution failed
