"""Pins the conforming ground-truth fixtures (tests/golden/make_conforming.py,
reference ``qttfem.oracle.ConformingSystem`` + splu) against the oracle's QTT
pipeline (oracle/fem.py assemble -> concat -> dirichlet, dense solve) at d=4:
configs 1, 4 (variable E, SURVEY §8(c) extension on both sides) and 5
(L-shape, penalty coupling vs merged nodes)."""

import os

import numpy as np
import pytest

from oracle import fem as F
from oracle import tt as O
from paper_2501_07778_b200.configs import config
from paper_2501_07778_b200.topology import DomainTopology

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("idx,tol", [(1, 1e-10), (4, 1e-10), (5, 1e-9)])
def test_conforming_fixture_matches_oracle_pipeline(idx, tol):
    meshes, mat, body, _ = config(idx, 4)
    topo = DomainTopology.from_subdomains(meshes)
    systems = F.assemble_all(meshes, mat, "zorder", 1e-13, body)
    K, f, mask, g = F.concat(systems, topo, eps=1e-13)
    K, f = F.dirichlet(K, f, mask, g, eps=1e-13)
    u = np.linalg.solve(O.full(K), O.full(f))
    z = np.load(os.path.join(GOLD, f"conforming_c{idx}_d4.npz"))
    uc = O.full([z[f"cores_{k}"] for k in range(len(z["ranks"]) - 1)])
    assert abs(np.linalg.norm(uc) - float(z["norm"])) <= 1e-12 * float(z["norm"])
    assert np.linalg.norm(u - uc) / np.linalg.norm(uc) <= tol
