"""Device element grids, QTT assembly, coupling and Dirichlet against the
reference's golden fixtures and the oracle."""

import os

import numpy as np
import pytest

from tests.golden import cases

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, f"{name}.npz"))


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def mesh_of(spec):
    from paper_2501_07778_b200.mesh import SubdomainMesh

    return SubdomainMesh(np.asarray(spec["corners"]), spec["d"], dict(spec.get("tags", {})),
                         dict(spec.get("tractions", {})))


def test_element_grids_golden():
    from paper_2501_07778_b200 import element as E
    from paper_2501_07778_b200.material import MaterialModel

    g = load("elements")
    for name, spec in cases.element_cases().items():
        mesh = mesh_of(spec)
        mat = MaterialModel(*spec["material"])
        kg = E.stiffness_value_grids(mesh, mat)
        gg = E.load_value_grid(mesh)
        for a in range(4):
            for b in range(4):
                assert rel(kg[(a, b)], g[f"{name}_K_{a}{b}"]) < 1e-14
                assert rel(gg[(a, b)], g[f"{name}_G_{a}{b}"]) < 1e-14


def test_shift_operators_golden():
    from paper_2501_07778_b200 import assembly as A
    from paper_2501_07778_b200.ttcore import tt_contract

    g = load("assembly")
    for name, (d, off) in cases.shift_cases().items():
        assert np.array_equal(tt_contract(A.qtt1d_shift(d, off)), g[f"shift_{name}"])


@pytest.mark.parametrize("name", list(cases.assembly_cases()))
def test_assembly_golden(name):
    from paper_2501_07778_b200 import assembly as A
    from paper_2501_07778_b200.material import MaterialModel
    from paper_2501_07778_b200.ttcore import tt_contract

    g = load("assembly")
    spec = cases.assembly_cases()[name]
    sysm = A.assemble_subdomain(mesh_of(spec), MaterialModel(*spec["material"]), spec["ordering"], spec["eps"],
                                body_force=spec["body"], cache=False)
    for blk in ("kxx", "kxy", "kyx", "kyy", "fx", "fy"):
        t = getattr(sysm, blk)
        assert t.ranks == tuple(g[f"{name}_{blk}_ranks"]), (blk, t.ranks)
        assert rel(tt_contract(t), g[f"{name}_{blk}"]) < 1e-11, blk


@pytest.mark.parametrize("name", ["single3", "lshape2", "cantilever2"])
def test_coupling_dirichlet_golden(name):
    from paper_2501_07778_b200 import assembly as A
    from paper_2501_07778_b200 import coupling as C
    from paper_2501_07778_b200.material import MaterialModel
    from paper_2501_07778_b200.topology import DomainTopology
    from paper_2501_07778_b200.ttcore import tt_contract

    g = load("coupling")
    spec = cases.coupling_cases()[name]
    meshes = [mesh_of(s) for s in spec["meshes"]]
    topo = DomainTopology.from_subdomains(meshes)
    mat = MaterialModel(*spec["material"])
    systems = [A.assemble_subdomain(m, mat, "zorder", spec["eps"], body_force=spec["body"]) for m in meshes]
    gs = C.concat_blocks(systems, topo, ordering="zorder", epsilon=spec["eps"])
    gd = C.apply_dirichlet(gs, epsilon=spec["eps"])
    assert abs(gs.gamma - g[f"{name}_gamma"]) < 1e-12 * gs.gamma
    for tag, t in (("K", gs.K), ("f", gs.f), ("mask", gs.mask), ("Kd", gd.K), ("fd", gd.f)):
        assert t.ranks == tuple(g[f"{name}_{tag}_ranks"]), (tag, t.ranks)
        assert rel(tt_contract(t), g[f"{name}_{tag}"]) < 1e-11, tag


def test_index_maps_golden():
    from paper_2501_07778_b200 import indexing as I

    g = load("index_maps")
    for d in (1, 2, 3, 4):
        assert np.array_equal(I.zorder_permutation(d), g[f"zperm_{d}"])
        assert np.array_equal(I.zorder_dof_permutation(d), g[f"zdof_{d}"])
    ii, jj = np.meshgrid(np.arange(8), np.arange(8), indexing="ij")
    assert np.array_equal(I.z_index(ii, jj, 3), g["z_index_3"])
    assert I.z_index(3, 2, 2) == 13
    assert I.canonical_index(2, 1, 2) == 6
    assert I.zorder_permutation(2)[13] == 11
    i, j = I.deinterleave(g["z_index_3"], 3)
    assert np.array_equal(i, ii) and np.array_equal(j, jj)
    with pytest.raises(ValueError):
        I.z_index(8, 0, 3)


@pytest.mark.parametrize("name", list(cases.round_cases()))
def test_round_golden(name):
    from paper_2501_07778_b200 import ttcore as T

    g = load("tt_ops")
    t, eps = cases.round_cases()[name]
    obj = T.TTVector(t) if t[0].ndim == 3 else T.TTMatrix(t)
    r = T.tt_round(obj, eps)
    assert r.ranks == tuple(g[f"round_{name}_ranks"])
    assert rel(T.tt_contract(r), g[f"round_{name}_dense"]) < max(eps, 1e-12)


@pytest.mark.parametrize("name", list(cases.decompose_cases()))
def test_decompose_golden(name):
    from paper_2501_07778_b200 import ttcore as T

    g = load("tt_ops")
    v, eps = cases.decompose_cases()[name]
    t = T.tt_decompose(v, eps)
    if eps > 0:
        assert t.ranks == tuple(g[f"decomp_{name}_ranks"])
    assert rel(T.tt_contract(t), g[f"decomp_{name}_dense"]) < max(eps, 1e-13)


def test_tt_ops_golden():
    from paper_2501_07778_b200 import solver as S
    from paper_2501_07778_b200 import ttcore as T

    g = load("tt_ops")
    for name, (A, x, B, y) in cases.tt_cases().items():
        TA, TB, tx, ty = T.TTMatrix(A), T.TTMatrix(B), T.TTVector(x), T.TTVector(y)
        assert rel(T.tt_contract(T.tt_matvec(TA, tx)), g[f"{name}_matvec"]) < 1e-13
        assert rel(T.tt_contract(T.tt_matmat(TA, TB)), g[f"{name}_matmat"]) < 1e-13
        assert rel(T.tt_contract(T.tt_add(tx, ty)), g[f"{name}_add"]) < 1e-14
        assert rel(T.tt_contract(T.tt_hadamard(tx, ty)), g[f"{name}_hadamard"]) < 1e-14
        assert abs(T.tt_norm(tx) - g[f"{name}_norm"]) <= 1e-13 * g[f"{name}_norm"]
        assert abs(T.tt_dot(tx, ty) - g[f"{name}_dot"]) <= 1e-12 * T.tt_norm(tx) * T.tt_norm(ty)
    out = S.apply_tt_matrix(T.TTMatrix(cases.apply_case()), g["apply_v"])
    assert isinstance(out, np.ndarray) and rel(out, g["apply_out"]) < 1e-13


@pytest.mark.parametrize("d", [3, 4])
def test_variable_modulus_assembly_matches_oracle(d):
    """Config-4 extension (E(x,y) at the Gauss points): device assembly vs the
    oracle restatement (itself pinned by tests/test_oracle_config4.py)."""
    from oracle import fem as F
    from oracle import tt as O
    from paper_2501_07778_b200 import assembly as A
    from paper_2501_07778_b200.material import MaterialModel, config4_modulus
    from paper_2501_07778_b200.mesh import SubdomainMesh
    from paper_2501_07778_b200.ttcore import tt_contract

    unit = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
    mat = MaterialModel(1.0, 0.3, "plane-stress", modulus_field=config4_modulus)
    mesh = SubdomainMesh(unit, d, {"left": "clamped"})
    ref = F.assemble(mesh, mat, "zorder", 1e-10, body=(0.0, -1.0))
    got = A.assemble_subdomain(mesh, mat, "zorder", 1e-10, body_force=(0.0, -1.0), cache=False)
    for blk in ("kxx", "kxy", "kyx", "kyy", "fx", "fy"):
        t = getattr(got, blk)
        assert t.ranks == O.ranks(ref[blk]), (blk, t.ranks, O.ranks(ref[blk]))
        assert rel(tt_contract(t), O.full(ref[blk])) < 1e-9, blk


@pytest.mark.parametrize("ordering,paper_det", [("canonical", False), ("canonical", True), ("zorder", True)])
def test_general_quad_orderings_match_oracle(ordering, paper_det):
    """Secondary API surface: canonical node ordering and
    the paper's determinant variant on a non-parallelogram patch (general
    element grids, assembly.py:131-158, element.py:95-100) against the
    oracle restatement; identical ranks, dense agreement."""
    from oracle import fem as F
    from oracle import tt as O
    from paper_2501_07778_b200 import assembly as A
    from paper_2501_07778_b200.material import MaterialModel
    from paper_2501_07778_b200.mesh import SubdomainMesh
    from paper_2501_07778_b200.ttcore import tt_contract

    quad = np.array([[0.0, 0.0], [1.2, 0.1], [1.0, 0.9], [-0.1, 1.1]])
    mat = MaterialModel(2.0, 0.25, "plane-strain")
    mesh = SubdomainMesh(quad, 3, {"left": "clamped"}, {"right": (0.5, -1.0)})
    ref = F.assemble(mesh, mat, ordering, 1e-11, body=(0.3, -1.0), paper_det=paper_det)
    got = A.assemble_subdomain(mesh, mat, ordering, 1e-11, body_force=(0.3, -1.0),
                               paper_determinant=paper_det, cache=False)
    for blk in ("kxx", "kxy", "kyx", "kyy"):
        t = getattr(got, blk)
        assert t.ranks == O.ranks(ref[blk]), (blk, t.ranks, O.ranks(ref[blk]))
        assert rel(tt_contract(t), O.full(ref[blk])) < 1e-9, blk
