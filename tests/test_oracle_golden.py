"""Pin the CPU oracle (oracle/) to golden vectors produced by the reference
itself (tests/golden/make_golden.py).  CPU only."""

import os

import numpy as np
import pytest

from oracle import fem as F
from oracle import tt as O
from paper_2501_07778_b200.material import MaterialModel
from paper_2501_07778_b200.mesh import SubdomainMesh
from paper_2501_07778_b200.topology import DomainTopology
from tests.golden import cases

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, f"{name}.npz"))


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def mesh_of(spec):
    return SubdomainMesh(np.asarray(spec["corners"]), spec["d"], dict(spec.get("tags", {})),
                         dict(spec.get("tractions", {})))


def test_tt_ops_golden():
    g = load("tt_ops")
    for name, (A, x, B, y) in cases.tt_cases().items():
        assert rel(O.full(O.matvec(A, x)), g[f"{name}_matvec"]) < 1e-13
        assert rel(O.full(O.matmat(A, B)), g[f"{name}_matmat"]) < 1e-13
        assert rel(O.full(O.add(x, y)), g[f"{name}_add"]) < 1e-14
        assert rel(O.full(O.hadamard(x, y)), g[f"{name}_hadamard"]) < 1e-14
        assert abs(O.norm(x) - g[f"{name}_norm"]) <= 1e-13 * g[f"{name}_norm"]
        assert abs(O.dot(x, y) - g[f"{name}_dot"]) <= 1e-12 * O.norm(x) * O.norm(y)
    A = cases.apply_case()
    assert rel(O.apply_dense(A, g["apply_v"]), g["apply_out"]) < 1e-13


@pytest.mark.parametrize("name", list(cases.round_cases()))
def test_round_golden(name):
    g = load("tt_ops")
    t, eps = cases.round_cases()[name]
    r = O.round_tt(t, eps)
    assert O.ranks(r) == tuple(g[f"round_{name}_ranks"])
    assert rel(O.full(r), g[f"round_{name}_dense"]) < max(eps, 1e-12)


@pytest.mark.parametrize("name", list(cases.decompose_cases()))
def test_decompose_golden(name):
    g = load("tt_ops")
    v, eps = cases.decompose_cases()[name]
    t = O.decompose_vector(v, eps)
    assert O.ranks(t) == tuple(g[f"decomp_{name}_ranks"])
    assert rel(O.full(t), g[f"decomp_{name}_dense"]) < max(eps, 1e-13)


def test_index_maps_golden():
    g = load("index_maps")
    for d in (1, 2, 3, 4):
        assert np.array_equal(O.zorder_permutation(d), g[f"zperm_{d}"])
        assert np.array_equal(O.zorder_dof_permutation(d), g[f"zdof_{d}"])
    ii, jj = np.meshgrid(np.arange(8), np.arange(8), indexing="ij")
    assert np.array_equal(O.z_index(ii, jj, 3), g["z_index_3"])
    # known answers (test_indexing.py:24-41)
    assert O.z_index(3, 2, 2) == 13
    assert O.zorder_permutation(2)[13] == 11


def test_element_grids_golden():
    g = load("elements")
    for name, spec in cases.element_cases().items():
        mesh = mesh_of(spec)
        mat = MaterialModel(*spec["material"])
        for a in range(4):
            for b in range(4):
                assert rel(F.stiffness_grid(mesh, mat, a, b), g[f"{name}_K_{a}{b}"]) < 1e-14
                assert rel(F.load_grid(mesh, a, b), g[f"{name}_G_{a}{b}"]) < 1e-14


def test_shift_operators_golden():
    g = load("assembly")
    for name, (d, off) in cases.shift_cases().items():
        assert np.array_equal(O.full(F.shift1d(d, off)), g[f"shift_{name}"])


@pytest.mark.parametrize("name", list(cases.assembly_cases()))
def test_assembly_golden(name):
    g = load("assembly")
    spec = cases.assembly_cases()[name]
    mesh = mesh_of(spec)
    sysd = F.assemble(mesh, MaterialModel(*spec["material"]), spec["ordering"], spec["eps"], body=spec["body"])
    for blk in ("kxx", "kxy", "kyx", "kyy", "fx", "fy"):
        assert O.ranks(sysd[blk]) == tuple(g[f"{name}_{blk}_ranks"]), blk
        assert rel(O.full(sysd[blk]), g[f"{name}_{blk}"]) < 1e-11, blk


@pytest.mark.parametrize("name", ["single3", "lshape2", "cantilever2"])
def test_coupling_golden(name):
    g = load("coupling")
    spec = cases.coupling_cases()[name]
    meshes = [mesh_of(s) for s in spec["meshes"]]
    topo = DomainTopology.from_subdomains(meshes)
    mat = MaterialModel(*spec["material"])
    systems = F.assemble_all(meshes, mat, "zorder", spec["eps"], spec["body"])
    K, f, tau, gam = F.concat(systems, topo, None, "zorder", spec["eps"])
    Kd, fd = F.dirichlet(K, f, tau, gam, None, spec["eps"])
    assert abs(gam - g[f"{name}_gamma"]) < 1e-12 * gam
    for tag, t in (("K", K), ("f", f), ("mask", tau), ("Kd", Kd), ("fd", fd)):
        assert O.ranks(t) == tuple(g[f"{name}_{tag}_ranks"]), tag
        assert rel(O.full(t), g[f"{name}_{tag}"]) < 1e-11, tag


@pytest.mark.parametrize("name", ["single3", "lshape2", "cantilever2"])
def test_oracle_amen_matches_reference_solution(name):
    from oracle import amen

    g = load("coupling")
    spec = cases.coupling_cases()[name]
    meshes = [mesh_of(s) for s in spec["meshes"]]
    topo = DomainTopology.from_subdomains(meshes)
    mat = MaterialModel(*spec["material"])
    systems = F.assemble_all(meshes, mat, "zorder", spec["eps"], spec["body"])
    K, f, tau, gam = F.concat(systems, topo, None, "zorder", spec["eps"])
    Kd, fd = F.dirichlet(K, f, tau, gam, None, spec["eps"])
    out = amen.solve(Kd, fd, eps=spec["solve"], seed=0)
    assert out["converged"]
    kd, fdd = g[f"{name}_Kd"], g[f"{name}_fd"]
    u_exact = np.linalg.solve(kd, fdd)
    err = rel(O.full(out["u"]), u_exact)
    ref_err = rel(g[f"{name}_u"], u_exact)
    assert err <= max(10 * ref_err, np.linalg.cond(kd) * spec["solve"]) + 1e-10
