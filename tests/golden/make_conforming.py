"""Conforming ground truth for the BASELINE solves.

Runs the REFERENCE's independent sparse conforming FEM
(``qttfem.oracle.ConformingSystem``, oracle.py:148-325: merged node ids,
direct per-element Jacobians, COO->CSR scatter, Dirichlet elimination) and
solves it with ``scipy.sparse.linalg.splu`` directly (pyamg, which the
reference uses above 700k DoFs (oracle.py:268-294), is not installed; the
6.3M-DoF L-shape does not fit one SuperLU factorisation and goes through
per-patch LUs + an interface Schur complement, ``schur_solve``).  Run in the
development container only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_conforming.py 4 10
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_conforming.py 5 10

The solution is scattered into the QTT global layout of the coupled system
(flat = Z(i, j) + 4^d (m + q_pad c), coupling.py:1-13,256-296; padded
subdomain slots are zero) and stored as a TT compressed with the reference's
own ``tt_decompose`` at eps = 1e-12 (a few MB instead of 16-64 MB of dense
vector; the 1e-12 compression error is far below the 1e-8 gate).  Stored:
``cores_*``, ``ranks``, ``norm`` (exact 2-norm of the dense vector),
``compress_err`` (dense relative error of the stored TT), sampled entries,
and the splu residual.

Config 4's spatially varying modulus (SURVEY §8(c) extension) has no
reference support: the element loop of ``_element_matrices``
(oracle.py:53-108) is restated here with the integrand multiplied by
E(x_g, y_g) at the physical Gauss point, and the parallelogram shortcut
(oracle.py:174-180) is bypassed, exactly as SURVEY §8(c) prescribes.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import qttfem.oracle as RO  # noqa: E402
from qttfem.element import quadrature_rule, shape_functions  # noqa: E402
from qttfem.indexing import z_index  # noqa: E402
from qttfem.material import MaterialModel as RMat  # noqa: E402
from qttfem.mesh import SubdomainMesh as RMesh  # noqa: E402
from qttfem.topology import DomainTopology as RTopo  # noqa: E402
from qttfem.ttcore import tt_contract, tt_decompose  # noqa: E402
from scipy.sparse import linalg as spla  # noqa: E402

UNIT = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])


def modulus(x, y):
    """BASELINE config 4: E(x, y) = 1 + 0.5 sin(2 pi x) sin(2 pi y)."""
    return 1.0 + 0.5 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y)


def element_matrices_var_e(mesh, material, quadrature):
    """(ne, ne, 4, 4, 2, 2) stiffness with E at the physical Gauss point and
    the (unweighted) mass grid; same index conventions as oracle.py:53-108."""
    coords = mesh.node_coords()
    ec = np.stack([coords[:-1, :-1], coords[1:, :-1], coords[1:, 1:], coords[:-1, 1:]], axis=2)
    ne = mesh.n_elem
    C = material.C
    pts, wts = quadrature_rule(quadrature)
    ke = np.zeros((ne, ne, 4, 4, 2, 2))
    me = np.zeros((ne, ne, 4, 4))
    for gx, wx in zip(pts, wts):
        for gy, wy in zip(pts, wts):
            vals, grads = shape_functions(gx, gy)
            jac = np.einsum("kr,ijkc->ijrc", grads, ec)
            det = jac[..., 0, 0] * jac[..., 1, 1] - jac[..., 0, 1] * jac[..., 1, 0]
            pos = np.einsum("k,ijkc->ijc", vals, ec)
            e = modulus(pos[..., 0], pos[..., 1])
            # physical gradients: (4, ne, ne)
            gxs = (grads[:, 0, None, None] * jac[None, ..., 1, 1] - grads[:, 1, None, None] * jac[None, ..., 0, 1]) / det
            gys = (-grads[:, 0, None, None] * jac[None, ..., 1, 0] + grads[:, 1, None, None] * jac[None, ..., 0, 0]) / det
            w = wx * wy * det
            we = w * e
            for a in range(4):
                for b in range(4):
                    ke[:, :, a, b, 0, 0] += we * (C[0, 0] * gxs[a] * gxs[b] + C[2, 2] * gys[a] * gys[b])
                    ke[:, :, a, b, 0, 1] += we * (C[0, 1] * gxs[a] * gys[b] + C[2, 2] * gys[a] * gxs[b])
                    ke[:, :, a, b, 1, 0] += we * (C[0, 1] * gys[a] * gxs[b] + C[2, 2] * gxs[a] * gys[b])
                    ke[:, :, a, b, 1, 1] += we * (C[1, 1] * gys[a] * gys[b] + C[2, 2] * gxs[a] * gxs[b])
                    me[:, :, a, b] += w * vals[a] * vals[b]
    return ke, me


def problem(idx: int, d: int):
    if idx == 4:
        meshes = [RMesh(UNIT, d, {"left": "clamped"}, {"right": (1.0, 0.0)})]
        return meshes, RMat(1.0, 0.3, "plane-stress"), (0.0, 0.0), True
    if idx == 40:  # constant-E variant of config 4 (SURVEY's config-4-like probe)
        meshes = [RMesh(UNIT, d, {"left": "clamped"}, {"right": (1.0, 0.0)})]
        return meshes, RMat(1.0, 0.3, "plane-stress"), (0.0, 0.0), False
    if idx == 5:
        meshes = [RMesh(UNIT, d), RMesh(UNIT + [1.0, 0.0], d), RMesh(UNIT + [0.0, 1.0], d, {"top": "clamped"})]
        return meshes, RMat(1.0, 0.3, "plane-strain"), (0.0, -1.0), False
    if idx == 1:
        meshes = [RMesh(UNIT, d, {"left": "clamped"})]
        return meshes, RMat(1.0, 0.3, "plane-stress"), (0.0, -1.0), False
    raise ValueError(idx)


class _NotParallelogram:
    """Mesh proxy that forces the per-element path (oracle.py:181-184)."""

    def __init__(self, mesh):
        self._m = mesh

    def __getattr__(self, name):
        return getattr(self._m, name)

    def is_parallelogram(self):
        return False


def schur_solve(system, free, kff, ff, tol=1e-15, maxit=3000):
    """Direct solve of the merged multi-patch system when one sparse LU of
    the whole system does not fit (SuperLU runs out of memory at 6.3M DoFs):
    the DoFs of nodes shared by two or more patches form the interface set G;
    every patch's remaining DoFs are factorised on their own (each block is
    nonsingular: removing the interface DoFs pins the patch), and the
    interface Schur complement S = K_GG - sum_m K_Gm K_mm^-1 K_mG (SPD) is
    solved by conjugate gradients to ~1e-15, then the patch DoFs are
    back-substituted.  Finished by one step of iterative refinement on the
    full system."""
    nodes_of = system.node_ids
    q = nodes_of.shape[0]
    count = np.zeros(system.n_nodes, dtype=np.int64)
    for m in range(q):
        count[np.unique(nodes_of[m])] += 1
    owner = np.full(system.n_nodes, -1, dtype=np.int64)
    for m in range(q):
        ids = np.unique(nodes_of[m])
        owner[ids[count[ids] == 1]] = m
    dof_owner = np.repeat(owner, 2)[free]  # -1: interface
    G = np.flatnonzero(dof_owner < 0)
    blocks = []
    for m in range(q):
        I = np.flatnonzero(dof_owner == m)
        t0 = time.perf_counter()
        lu = spla.splu(kff[I][:, I].tocsc(), permc_spec="MMD_AT_PLUS_A")
        print(f"  patch {m}: {I.size} dofs factorised in {time.perf_counter() - t0:.1f}s", flush=True)
        blocks.append((I, lu, kff[I][:, G].tocsr(), kff[G][:, I].tocsr()))
    kgg = kff[G][:, G].tocsr()

    def solve_full(b):
        bg = b[G].copy()
        ys = []
        for I, lu, kig, kgi in blocks:
            y = lu.solve(b[I])
            ys.append(y)
            bg -= kgi @ y

        def S(v):
            out = kgg @ v
            for I, lu, kig, kgi in blocks:
                out -= kgi @ lu.solve(kig @ v)
            return out

        # conjugate gradients on the SPD Schur complement
        x = np.zeros_like(bg)
        r = bg.copy()
        p = r.copy()
        rr = r @ r
        nb = np.sqrt(bg @ bg)
        t0 = time.perf_counter()
        for it in range(maxit):
            if it % 50 == 0:
                print(f"    CG it {it} res {np.sqrt(rr) / nb:.2e} t {time.perf_counter() - t0:.0f}s", flush=True)
            Sp = S(p)
            a = rr / (p @ Sp)
            x += a * p
            r -= a * Sp
            rr_new = r @ r
            if np.sqrt(rr_new) <= tol * nb:
                break
            p = r + (rr_new / rr) * p
            rr = rr_new
        print(f"  schur CG: {it + 1} iterations, residual {np.sqrt(rr_new) / nb:.2e}", flush=True)
        out = np.zeros_like(b)
        out[G] = x
        for (I, lu, kig, kgi), y in zip(blocks, ys):
            out[I] = y - lu.solve(kig @ x)
        return out

    u = solve_full(ff)
    r = ff - kff @ u
    print(f"  residual before refinement {np.linalg.norm(r) / np.linalg.norm(ff):.2e}", flush=True)
    return u + solve_full(r)


def main(idx: int, d: int):
    meshes, mat, body, var_e = problem(idx, d)
    topo = RTopo.from_subdomains(meshes)
    t0 = time.perf_counter()
    if var_e:
        RO._element_matrices = element_matrices_var_e
        topo.subdomains[:] = [_NotParallelogram(m) for m in topo.subdomains]
    system = RO.ConformingSystem(topo, mat, body)
    t1 = time.perf_counter()
    free = ~system.constrained
    kff = system.K[free][:, free].tocsr()
    ff = system.f[free]
    if topo.q == 1 or free.sum() <= 2_500_000:
        uf = spla.splu(kff.tocsc(), permc_spec="MMD_AT_PLUS_A").solve(ff)
    else:
        uf = schur_solve(system, free, kff, ff)
    res = float(np.linalg.norm(kff @ uf - ff) / np.linalg.norm(ff))
    t2 = time.perf_counter()
    u = np.zeros(system.n_dofs)
    u[free] = uf
    q = topo.q
    s = 0 if q == 1 else int(np.ceil(np.log2(q)))
    qp = 1 << s
    n = 1 << d
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    z = z_index(ii, jj, d)
    flat = np.zeros(2 * qp * 4**d)
    for m in range(q):
        ids = system.node_ids[m]
        for c in range(2):
            flat[z + 4**d * (m + qp * c)] = u[2 * ids + c]
    t3 = time.perf_counter()
    tt = tt_decompose(flat, 1e-12)
    back = tt_contract(tt)
    cerr = float(np.linalg.norm(back - flat) / np.linalg.norm(flat))
    t4 = time.perf_counter()
    rng = np.random.default_rng(7)
    idxs = np.sort(rng.choice(flat.size, 256, replace=False))
    out = {f"cores_{k}": c for k, c in enumerate(tt.cores)}
    out.update(
        ranks=np.asarray(tt.ranks, dtype=np.int64),
        norm=np.array(np.linalg.norm(flat)),
        compress_err=np.array(cerr),
        sample_idx=idxs.astype(np.int64),
        sample_val=flat[idxs],
        splu_residual=np.array(res),
        n_free=np.array(int(free.sum())),
        d=np.array(d),
    )
    path = os.path.join(HERE, f"conforming_c{idx}_d{d}.npz")
    np.savez_compressed(path, **out)
    print(f"config {idx} d={d}: dofs {system.n_dofs} free {int(free.sum())} assembly {t1 - t0:.1f}s "
          f"splu {t2 - t1:.1f}s residual {res:.2e} tt ranks max {max(tt.ranks)} compress err {cerr:.2e} "
          f"({t4 - t3:.1f}s) -> {path} ({os.path.getsize(path) / 1e6:.1f} MB)", flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]))
