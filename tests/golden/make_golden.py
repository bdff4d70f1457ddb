"""Generate golden fixtures by running the REFERENCE implementation.

Run in the development container (the reference is importable there,
read-only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.npz.  The GPU box never reads /root/reference; tests
only load these files.  Inputs are seeded so the same arrays can be rebuilt
by the tests (see tests/golden/cases.py).

Reference quirk handled here: ``concat_blocks`` caches Pi*K products under
``(id(pi), id(blk))`` (coupling.py:404-409) where ``pi`` is a temporary; when
CPython reuses the freed id the cache returns a product of the WRONG
connectivity operator (observed: 28% relative error in K for the L-shape at
d=3).  The fixtures are generated with the connectivity operators kept alive
(so ids stay unique), which is the reference's intended behaviour.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import qttfem.assembly as RA  # noqa: E402
import qttfem.coupling as RC  # noqa: E402
import qttfem.element as RE  # noqa: E402
import qttfem.indexing as RI  # noqa: E402
import qttfem.solver as RS  # noqa: E402
import qttfem.ttcore as RT  # noqa: E402
from qttfem.material import MaterialModel as RMat  # noqa: E402
from qttfem.mesh import SubdomainMesh as RMesh  # noqa: E402
from qttfem.topology import DomainTopology as RTopo  # noqa: E402

from tests.golden import cases  # noqa: E402

_alive = []
_orig_bc = RC.build_connectivity


def _bc(*a, **k):
    r = _orig_bc(*a, **k)
    _alive.append(r)
    return r


RC.build_connectivity = _bc


def _ranks(t):
    return np.asarray(t.ranks, dtype=np.int64)


def tt_ops():
    out = {}
    for name, (A, x, B, y) in cases.tt_cases().items():
        TA, TB = RT.TTMatrix(A), RT.TTMatrix(B)
        tx, ty = RT.TTVector(x), RT.TTVector(y)
        out[f"{name}_matvec"] = RT.tt_contract(RT.tt_matvec(TA, tx))
        out[f"{name}_matmat"] = RT.tt_contract(RT.tt_matmat(TA, TB))
        out[f"{name}_add"] = RT.tt_contract(RT.tt_add(tx, ty))
        out[f"{name}_hadamard"] = RT.tt_contract(RT.tt_hadamard(tx, ty))
        out[f"{name}_norm"] = np.array(RT.tt_norm(tx))
        out[f"{name}_dot"] = np.array(RT.tt_dot(tx, ty))
    for name, (t, eps) in cases.round_cases().items():
        r = RT.tt_round(RT.TTVector(t) if t[0].ndim == 3 else RT.TTMatrix(t), eps)
        out[f"round_{name}_ranks"] = _ranks(r)
        out[f"round_{name}_dense"] = RT.tt_contract(r)
    for name, (v, eps) in cases.decompose_cases().items():
        t = RT.tt_decompose(v, eps)
        out[f"decomp_{name}_ranks"] = _ranks(t)
        out[f"decomp_{name}_dense"] = RT.tt_contract(t)
    A = cases.apply_case()
    v = np.random.default_rng(77).standard_normal(RT.TTMatrix(A).shape[1])
    out["apply_v"] = v
    out["apply_out"] = RS.apply_tt_matrix(RT.TTMatrix(A), v)
    return out


def index_maps():
    out = {}
    for d in (1, 2, 3, 4):
        out[f"zperm_{d}"] = RI.zorder_permutation(d)
        out[f"zdof_{d}"] = RI.zorder_dof_permutation(d)
    ii, jj = np.meshgrid(np.arange(8), np.arange(8), indexing="ij")
    out["z_index_3"] = RI.z_index(ii, jj, 3)
    return out


def _rmesh(spec):
    return RMesh(np.asarray(spec["corners"]), spec["d"], dict(spec.get("tags", {})),
                 dict(spec.get("tractions", {})))


def elements():
    out = {}
    for name, spec in cases.element_cases().items():
        mesh = _rmesh(spec)
        mat = RMat(*spec["material"])
        for a in range(4):
            for b in range(4):
                out[f"{name}_K_{a}{b}"] = RE.element_stiffness_block(mesh, mat, RE.CORNERS[a], RE.CORNERS[b])
                out[f"{name}_G_{a}{b}"] = RE.element_load_block(mesh, RE.CORNERS[a], RE.CORNERS[b])
    return out


def assembly():
    out = {}
    for name, spec in cases.assembly_cases().items():
        mesh = _rmesh(spec)
        sysm = RA.assemble_subdomain(mesh, RMat(*spec["material"]), spec["ordering"], spec["eps"],
                                     body_force=spec["body"], cache=False)
        for blk in ("kxx", "kxy", "kyx", "kyy", "fx", "fy"):
            t = getattr(sysm, blk)
            out[f"{name}_{blk}"] = RT.tt_contract(t)
            out[f"{name}_{blk}_ranks"] = _ranks(t)
    for name, (d, offset) in cases.shift_cases().items():
        out[f"shift_{name}"] = RT.tt_contract(RA.qtt1d_shift(d, offset))
    return out


def coupling():
    out = {}
    for name, spec in cases.coupling_cases().items():
        meshes = [_rmesh(s) for s in spec["meshes"]]
        topo = RTopo.from_subdomains(meshes)
        mat = RMat(*spec["material"])
        systems = [RA.assemble_subdomain(m, mat, "zorder", spec["eps"], body_force=spec["body"]) for m in meshes]
        g = RC.concat_blocks(systems, topo, ordering="zorder", epsilon=spec["eps"])
        g2 = RC.apply_dirichlet(g, epsilon=spec["eps"])
        out[f"{name}_gamma"] = np.array(g.gamma)
        for tag, t in (("K", g.K), ("f", g.f), ("mask", g.mask), ("Kd", g2.K), ("fd", g2.f)):
            out[f"{name}_{tag}"] = RT.tt_contract(t)
            out[f"{name}_{tag}_ranks"] = _ranks(t)
        if spec.get("solve"):
            res = RS.solve(g2.K, g2.f, RS.SolverConfig(epsilon=spec["solve"], seed=0, local_solver="direct"))
            out[f"{name}_u"] = RT.tt_contract(res.u)
            out[f"{name}_u_ranks"] = _ranks(res.u)
            out[f"{name}_residual"] = np.array(res.residual)
    return out


def main():
    for fname, fn in (("tt_ops", tt_ops), ("index_maps", index_maps), ("elements", elements),
                      ("assembly", assembly), ("coupling", coupling)):
        data = fn()
        np.savez_compressed(os.path.join(HERE, f"{fname}.npz"), **data)
        size = os.path.getsize(os.path.join(HERE, f"{fname}.npz"))
        print(f"{fname}.npz: {len(data)} arrays, {size / 1e3:.1f} kB")


if __name__ == "__main__":
    main()
