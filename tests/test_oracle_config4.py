"""Pins the oracle's config-4 extension (spatially varying Young's modulus,
SURVEY.md §8(c)) that no reference test covers: the QTT stiffness assembled
by oracle/fem.py with ``modulus_field`` must equal a conventional
element-by-element Q1 assembly (2x2 Gauss, E evaluated at the physical Gauss
points) written independently here, node-for-node in Z order."""

import numpy as np
import pytest

from oracle import fem as F
from oracle import tt as O
from paper_2501_07778_b200.material import MaterialModel, config4_modulus
from paper_2501_07778_b200.mesh import SubdomainMesh

UNIT = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])


def _element_loop(d, mat, corners):
    """Dense global stiffness, DoF = 2 * (i + n j) + c (i: x node index)."""
    n = 1 << d
    C = mat.C
    a = 1.0 / np.sqrt(3.0)
    K = np.zeros((2 * n * n, 2 * n * n))
    for ej in range(n - 1):
        for ei in range(n - 1):
            nodes = [(ei, ej), (ei + 1, ej), (ei + 1, ej + 1), (ei, ej + 1)]  # element.py:30 corner order
            xy = np.array([corners_map(corners, i / (n - 1), j / (n - 1)) for i, j in nodes])
            ke = np.zeros((8, 8))
            for gx in (-a, a):
                for gy in (-a, a):
                    v, g = F.shape(gx, gy)
                    J = g.T @ xy  # rows: d/dxi, d/deta
                    det = np.linalg.det(J)
                    dN = np.linalg.solve(J, g.T).T  # (4, 2) physical gradients
                    B = np.zeros((3, 8))
                    B[0, 0::2] = dN[:, 0]
                    B[1, 1::2] = dN[:, 1]
                    B[2, 0::2] = dN[:, 1]
                    B[2, 1::2] = dN[:, 0]
                    px, py = v @ xy
                    e = mat.modulus_field(px, py) if mat.modulus_field is not None else 1.0
                    ke += e * det * (B.T @ C @ B)
            dofs = np.array([[2 * (i + n * j), 2 * (i + n * j) + 1] for i, j in nodes]).ravel()
            K[np.ix_(dofs, dofs)] += ke
    return K


def corners_map(corners, s, t):
    """Bilinear map of the unit square onto the patch (mesh.py bilinear map)."""
    c = np.asarray(corners, dtype=float)
    return (1 - s) * (1 - t) * c[0] + s * (1 - t) * c[1] + s * t * c[2] + (1 - s) * t * c[3]


@pytest.mark.parametrize("d", [2, 3])
def test_variable_modulus_assembly_matches_element_loop(d):
    mat = MaterialModel(1.0, 0.3, "plane-stress", modulus_field=config4_modulus)
    mesh = SubdomainMesh(UNIT, d, {"left": "clamped"})
    blocks = F.assemble(mesh, mat, "zorder", 1e-14)
    n = 1 << d
    z = np.array([O.z_index(i, j, d) for j in range(n) for i in range(n)])  # node i + n j -> Z
    ref = _element_loop(d, mat, UNIT)
    for (al, be), name in {(0, 0): "kxx", (0, 1): "kxy", (1, 0): "kyx", (1, 1): "kyy"}.items():
        qd = O.full(blocks[name])  # (4^d, 4^d) in Z order
        got = qd[np.ix_(z, z)]
        want = ref[al::2, be::2]
        assert np.linalg.norm(got - want) <= 1e-11 * np.linalg.norm(want), name


def test_element_loop_reduces_to_constant_modulus():
    """The same element loop with E = 1 reproduces the reference's
    constant-modulus shortcut path in the oracle (cross-check of the loop)."""
    d = 2
    mat = MaterialModel(1.0, 0.3, "plane-stress")
    mesh = SubdomainMesh(UNIT, d, {"left": "clamped"})
    blocks = F.assemble(mesh, mat, "zorder", 1e-14)
    n = 1 << d
    z = np.array([O.z_index(i, j, d) for j in range(n) for i in range(n)])
    ref = _element_loop(d, mat, UNIT)
    got = O.full(blocks["kxy"])[np.ix_(z, z)]
    assert np.linalg.norm(got - ref[0::2, 1::2]) <= 1e-11 * np.linalg.norm(ref[0::2, 1::2])
