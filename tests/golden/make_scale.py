"""Golden fixtures at BASELINE scale (VERDICT r1 "next" item 1).

Run in the development container (the reference is importable there):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_scale.py

Writes ``tests/golden/scale.npz``:

* ``c1_*`` — config 1 (d=5) by the REFERENCE: Dirichlet-conjugated global K
  and f cores (assemble_subdomain -> concat_blocks -> apply_dirichlet,
  eps=1e-8) and the converged solution of ``solve(SolverConfig(epsilon=1e-8,
  seed=0, local_solver="direct"))`` (solver.py:239-389) as a dense vector,
  with its ranks, sweep count and residual.
* ``c2_4x16_*`` — config 2 pair (rA, rx) = (4, 16) at d = 24 by the
  REFERENCE: ``tt_round(tt_matvec(A, x), 1e-10)`` cores and ranks.
* ``c3_*`` — config 3 by the REFERENCE: ranks of ``tt_round`` of the 16-term
  rank-128 sum at eps 1e-6 / 1e-10 and of ``tt_decompose`` of the 2^26 field.
* ``c4_*`` — config 4 (d=10, variable E) K and f cores assembled by the
  ORACLE (oracle/fem.py, the pinned restatement with the SURVEY §8(c)
  modulus extension, which the reference lacks).

Seeds follow SURVEY §8(d) (bench.make_inputs is the same generator).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import qttfem.assembly as RA  # noqa: E402
import qttfem.coupling as RC  # noqa: E402
import qttfem.solver as RS  # noqa: E402
import qttfem.ttcore as RT  # noqa: E402
from qttfem.indexing import z_index  # noqa: E402
from qttfem.material import MaterialModel as RMat  # noqa: E402
from qttfem.mesh import SubdomainMesh as RMesh  # noqa: E402
from qttfem.topology import DomainTopology as RTopo  # noqa: E402

UNIT = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])


def _put(out, prefix, t):
    for k, c in enumerate(t.cores):
        out[f"{prefix}_core{k}"] = np.asarray(c)
    out[f"{prefix}_ranks"] = np.asarray(t.ranks, dtype=np.int64)


def config1(out):
    mesh = RMesh(UNIT, 5, {"left": "clamped"})
    mat = RMat(1.0, 0.3, "plane-stress")
    sysm = RA.assemble_subdomain(mesh, mat, "zorder", 1e-8, body_force=(0.0, -1.0))
    topo = RTopo.from_subdomains([mesh])
    g = RC.apply_dirichlet(RC.concat_blocks([sysm], topo, ordering="zorder", epsilon=1e-8), epsilon=1e-8)
    _put(out, "c1_K", g.K)
    _put(out, "c1_f", g.f)
    t0 = time.perf_counter()
    res = RS.solve(g.K, g.f, RS.SolverConfig(epsilon=1e-8, seed=0, local_solver="direct"))
    print(f"config1 reference solve {time.perf_counter() - t0:.2f}s sweeps {res.sweeps} "
          f"residual {res.residual:.2e} ranks {res.u.ranks}", flush=True)
    out["c1_u"] = RT.tt_contract(res.u)
    out["c1_u_ranks"] = np.asarray(res.u.ranks, dtype=np.int64)
    out["c1_sweeps"] = np.array(res.sweeps)
    out["c1_residual"] = np.array(res.residual)


def config2(out):
    import bench

    A, x = bench.make_inputs(4, 16)
    t0 = time.perf_counter()
    z = RT.tt_round(RT.tt_matvec(RT.TTMatrix(A), RT.TTVector(x)), 1e-10)
    print(f"config2 (4,16) reference round {time.perf_counter() - t0:.2f}s ranks {z.ranks}", flush=True)
    _put(out, "c2_4x16_z", z)


def config3(out):
    rng = np.random.default_rng(3000)
    acc = None
    for _ in range(16):
        rk = [1] + [8] * 25 + [1]
        t = RT.TTVector([rng.standard_normal((rk[k], 2, rk[k + 1])) / np.sqrt(8) for k in range(26)])
        acc = t if acc is None else RT.tt_add(acc, t)
    for eps in (1e-6, 1e-10):
        out[f"c3_round_{eps:g}_ranks"] = np.asarray(RT.tt_round(acc, eps).ranks, dtype=np.int64)
    n = 1 << 13
    xs = np.arange(n) / (n - 1)
    X, Y = np.meshgrid(xs, xs, indexing="ij")
    g = np.sin(3 * X) * np.exp(-Y) + 0.1 * np.cos(7 * X * Y)
    v = np.empty(n * n)
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    v[z_index(ii, jj, 13)] = g
    t0 = time.perf_counter()
    tv = RT.tt_decompose(v, 1e-8)
    print(f"config3 reference TT-SVD {time.perf_counter() - t0:.2f}s ranks {tv.ranks}", flush=True)
    out["c3_ttsvd_ranks"] = np.asarray(tv.ranks, dtype=np.int64)


def config4(out, d=10):
    from oracle import fem as F
    from paper_2501_07778_b200.configs import config
    from paper_2501_07778_b200.topology import DomainTopology

    meshes, mat, body, eps = config(4, d)
    t0 = time.perf_counter()
    systems = F.assemble_all(meshes, mat, "zorder", eps, body)
    topo = DomainTopology.from_subdomains(meshes)
    K, f, mask, gamma = F.concat(systems, topo, eps=eps)
    K, f = F.dirichlet(K, f, mask, gamma, eps=eps)
    print(f"config4 d={d} oracle build {time.perf_counter() - t0:.1f}s K ranks {[c.shape[0] for c in K] + [1]}",
          flush=True)
    for k, c in enumerate(K):
        out[f"c4_K_core{k}"] = c
    for k, c in enumerate(f):
        out[f"c4_f_core{k}"] = c
    out["c4_d"] = np.array(d)
    out["c4_gamma"] = np.array(gamma)


def main():
    out = {}
    which = sys.argv[1:] or ["1", "2", "3", "4"]
    path = os.path.join(HERE, "scale.npz")
    if os.path.exists(path):
        old = np.load(path)
        out.update({k: old[k] for k in old.files})
    for w in which:
        {"1": config1, "2": config2, "3": config3, "4": config4}[w](out)
    np.savez_compressed(path, **out)
    print(f"scale.npz: {len(out)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
