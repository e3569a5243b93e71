"""TEST INFRASTRUCTURE ONLY — recipe that builds oracle/_ref from the reference.

The reference (flowbench 0.1.0) is pure Python + numba; "building" it means
installing the package from its own sources, unmodified, with pip (no index,
no dependency resolution: numpy / scipy / numba are in the image) into
`oracle/_ref/site`, and staging its own test modules in `oracle/_ref/tests`
so the GPU box -- where /root/reference does not exist -- can

* time the reference's own CPU path (bench.py --impl reference and the GPU
  line's cpu_baseline: stock `HelmholtzOperator.apply`, `cg` +
  `LORPreconditioner`, FLOWBENCH_BACKEND=numba, one core), and
* re-run the reference's operator / solver / Stokes tests against this
  package by import substitution (tests/test_reference_suite.py).

`oracle/_ref/` is git-ignored (no reference source enters the history) but
not gpurun-ignored, so it travels to the GPU box with the built .so.  Run by
`__graft_entry__.build()` whenever /root/reference is present:

    python oracle/build_ref.py [--force]
"""

import hashlib
import json
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PKG = "/root/reference/pkg"
OUT = os.path.join(HERE, "_ref")


def _digest(root):
    h = hashlib.sha256()
    for dp, dn, fn in sorted(os.walk(root)):
        dn.sort()
        for f in sorted(fn):
            if f.endswith(".py") or f.endswith(".toml"):
                p = os.path.join(dp, f)
                h.update(os.path.relpath(p, root).encode())
                with open(p, "rb") as fh:
                    h.update(fh.read())
    return h.hexdigest()


def build(force=False, quiet=True):
    """Returns the path of oracle/_ref, or None when the reference is absent."""
    if not os.path.isdir(REF_PKG):
        return OUT if os.path.isdir(os.path.join(OUT, "site", "flowbench")) else None
    digest = _digest(REF_PKG)
    info_path = os.path.join(OUT, "BUILD_INFO.json")
    if not force and os.path.exists(info_path):
        with open(info_path) as f:
            if json.load(f).get("sha256") == digest:
                return OUT
    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")  # the build writes egg-info next to the sources
        shutil.copytree(REF_PKG, src, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
               "--no-deps", "--no-compile", "--target", os.path.join(OUT, "site"), src]
        subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL if quiet else None,
                       stderr=subprocess.STDOUT if quiet else None)
    shutil.copytree(os.path.join(REF_PKG, "tests"), os.path.join(OUT, "tests"),
                    ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    with open(info_path, "w") as f:
        json.dump({"source": REF_PKG, "sha256": digest, "package": "flowbench 0.1.0",
                   "how": " ".join(cmd[1:])}, f, indent=1)
    return OUT


def site_path():
    """Directory to put on sys.path to import the reference `flowbench`."""
    p = os.path.join(OUT, "site")
    return p if os.path.isdir(os.path.join(p, "flowbench")) else None


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, quiet=False))
