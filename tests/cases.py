"""Shared fixtures: rebuild golden cases with the PRODUCT setup code."""

import json
import os

import numpy as np

from paper_1910_03032_b200 import geometry, spaces

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f)


def load(group):
    return np.load(os.path.join(GOLDEN, f"{group}.npz"))


def build(d, counts, periodic, perturb, p, vdim=1, seed=11):
    m = geometry.cartesian_mesh(tuple(counts), periodic=tuple(periodic) if periodic else None)
    if perturb:
        m = geometry.perturb_mesh(m, perturb, seed=seed)
    sp = spaces.FESpace(m, p, vdim=vdim)
    geom = geometry.compute_geometric_factors(m, sp.basis.quad)
    return m, sp, geom


def rel_err(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
