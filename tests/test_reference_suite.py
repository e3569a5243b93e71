"""The reference's own operator / solver / Stokes tests, run against this
package by import substitution (tests/refsuite/plugin.py).

The reference and its test modules come from oracle/_ref (built from
/root/reference by oracle/build_ref.py in the build container; it travels to
the GPU box).  Reference test files: pkg/tests/test_mfop.py,
test_solvers.py, test_stokes.py."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "oracle", "_ref", "tests")

# reference tests that exercise something other than this package's
# implementation (documented per test; everything else must pass)
NOT_APPLICABLE = {
}


@pytest.mark.gpu
@pytest.mark.parametrize("module", ["test_mfop.py", "test_solvers.py", "test_stokes.py",
                                    "test_lor.py"])
def test_reference_module_against_package(module):
    path = os.path.join(REF_TESTS, module)
    if not os.path.exists(path):
        pytest.skip("oracle/_ref not built (python oracle/build_ref.py needs /root/reference)")
    cmd = [sys.executable, "-m", "pytest", path, "-q", "-p", "tests.refsuite.plugin",
           "-p", "no:cacheprovider", "--rootdir", REF_TESTS, "-o", "addopts="]
    for t in NOT_APPLICABLE.get(module, {}):
        cmd += ["--deselect", f"{path}::{t}"]
    env = dict(os.environ, PYTHONPATH=ROOT)
    r = subprocess.run(cmd, cwd=ROOT, env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                       text=True, timeout=1500)
    tail = r.stdout[-3000:]
    assert r.returncode == 0, tail
    assert "libfbb200 kernel launches during the run: 0" not in r.stdout
    summary = [ln for ln in r.stdout.splitlines() if " passed" in ln]
    assert summary and "failed" not in summary[-1], tail
    print(f"{module}: {summary[-1].strip()}")
