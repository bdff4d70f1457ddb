"""Conforming ground truth for config 5 at d = 10 (6.3M DoFs), on the GPU box.

SuperLU cannot factorise the 6.3M-DoF L-shape (MemoryError in
make_conforming.py), so this generator restates the reference's conforming
oracle (qttfem/oracle.py:31-325) independently and solves it by
Jacobi-preconditioned conjugate gradients with torch sparse CSR products:

* nodes of the three patches are merged by their exact integer lattice
  coordinates (the union-find of tied pairs in oracle.py:31-50 merges the
  same nodes on this matching mesh);
* the Q1 element stiffness is the 2x2-Gauss integral of B^T C B (identical
  for every element of the axis-aligned unit patches, oracle.py:111-145);
* the consistent body-force load is sum_e int N_a b dA (oracle.py:202-206);
* clamped DoFs are eliminated (oracle.py:243-268).

It is test infrastructure only (not the product): it never touches the
package's kernels.  Validated against the reference-splu fixtures at d = 6
and d = 8 (``--check``).  Writes tests/golden/conforming_c5_d{d}_cg.npz in
the make_conforming.py format (QTT-layout solution compressed by the oracle's
TT-SVD at 1e-12).

    python tests/golden/make_conforming_gpu.py 10          # on the GPU box
    python tests/golden/make_conforming_gpu.py 8 --check   # vs splu fixture
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import tt as O  # noqa: E402

PATCH_OFFSETS = ((0, 0), (1, 0), (0, 1))  # UNIT, UNIT+[1,0], UNIT+[0,1]
E_MOD, NU = 1.0, 0.3
BODY = (0.0, -1.0)


def plane_strain_C(e, nu):
    lam = e * nu / ((1 + nu) * (1 - 2 * nu))
    mu = e / (2 * (1 + nu))
    return np.array([[lam + 2 * mu, lam, 0.0], [lam, lam + 2 * mu, 0.0], [0.0, 0.0, mu]])


def element_stiffness(h):
    """8x8 Q1 stiffness of an h x h square, DoF order (corner, component),
    corners CCW from the lower left (element.py:30)."""
    C = plane_strain_C(E_MOD, NU)
    g = 1.0 / np.sqrt(3.0)
    xy = np.array([[0, 0], [h, 0], [h, h], [0, h]], dtype=float)
    ke = np.zeros((8, 8))
    for xi in (-g, g):
        for eta in (-g, g):
            dn = 0.25 * np.array([[-(1 - eta), -(1 - xi)], [(1 - eta), -(1 + xi)],
                                  [(1 + eta), (1 + xi)], [-(1 + eta), (1 - xi)]])
            J = dn.T @ xy
            dN = np.linalg.solve(J, dn.T).T
            B = np.zeros((3, 8))
            B[0, 0::2] = dN[:, 0]
            B[1, 1::2] = dN[:, 1]
            B[2, 0::2] = dN[:, 1]
            B[2, 1::2] = dN[:, 0]
            ke += np.linalg.det(J) * (B.T @ C @ B)
    return ke


def assemble(d, dev):
    n = 1 << d
    h = 1.0 / (n - 1)
    # global lattice coordinates of every (patch, i, j) node
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    keys = []
    for ox, oy in PATCH_OFFSETS:
        I = ii + ox * (n - 1)
        J = jj + oy * (n - 1)
        keys.append(I.astype(np.int64) * (4 * n) + J.astype(np.int64))
    allk = np.stack(keys)  # (q, n, n)
    uniq, ids = np.unique(allk.ravel(), return_inverse=True)
    ids = ids.reshape(allk.shape)
    nn = uniq.size
    ke = torch.tensor(element_stiffness(h), device=dev)
    rows, cols, vals = [], [], []
    f = torch.zeros(2 * nn, dtype=torch.float64, device=dev)
    for m in range(len(PATCH_OFFSETS)):
        t = torch.tensor(ids[m], device=dev)
        cn = torch.stack([t[:-1, :-1], t[1:, :-1], t[1:, 1:], t[:-1, 1:]], dim=-1).reshape(-1, 4)
        dof = torch.stack([2 * cn, 2 * cn + 1], dim=-1).reshape(-1, 8)  # (ne, 8)
        rows.append(dof[:, :, None].expand(-1, 8, 8).reshape(-1))
        cols.append(dof[:, None, :].expand(-1, 8, 8).reshape(-1))
        vals.append(ke.reshape(1, 64).expand(dof.shape[0], 64).reshape(-1))
        load = h * h / 4.0  # int N_a dA over a square element
        for c in range(2):
            f.index_add_(0, (2 * cn + c).reshape(-1),
                         torch.full((cn.numel(),), load * BODY[c], dtype=torch.float64, device=dev))
    K = torch.sparse_coo_tensor(torch.stack([torch.cat(rows), torch.cat(cols)]), torch.cat(vals),
                                (2 * nn, 2 * nn)).coalesce()
    # clamp: top edge of patch 2
    clamp = np.unique(ids[2][:, n - 1])
    fixed = np.zeros(2 * nn, dtype=bool)
    fixed[2 * clamp] = True
    fixed[2 * clamp + 1] = True
    return K, f, fixed, ids, nn


def cg(K, b, tol=1e-15, maxit=400000, check_every=1000):
    Kc = K.to_sparse_csr()
    I, v = K.indices(), K.values()
    on = I[0] == I[1]
    diag = torch.zeros(K.shape[0], dtype=torch.float64, device=v.device).index_add_(0, I[0][on], v[on])
    dinv = 1.0 / diag
    x = torch.zeros_like(b)
    r = b.clone()
    z = dinv * r
    p = z.clone()
    rz = torch.dot(r, z)
    nb = torch.linalg.vector_norm(b)
    t0 = time.perf_counter()
    for it in range(maxit):
        Ap = torch.mv(Kc, p)
        a = rz / torch.dot(p, Ap)
        x += a * p
        r -= a * Ap
        if it % check_every == 0:
            rel = float(torch.linalg.vector_norm(r) / nb)
            print(f"  CG it {it} res {rel:.2e} t {time.perf_counter() - t0:.1f}s", flush=True)
            if rel <= tol:
                break
        z = dinv * r
        rz_new = torch.dot(r, z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    true = float(torch.linalg.vector_norm(b - torch.mv(Kc, x)) / nb)
    print(f"  CG done after {it + 1} iterations, true residual {true:.2e}", flush=True)
    return x, true


def main(d, check=False):
    dev = torch.device("cuda" if torch.cuda.is_available() else "cpu")
    t0 = time.perf_counter()
    K, f, fixed, ids, nn = assemble(d, dev)
    free = torch.tensor(~fixed, device=dev)
    idx = torch.nonzero(free).squeeze(1)
    pos = torch.full((2 * nn,), -1, dtype=torch.int64, device=dev)
    pos[idx] = torch.arange(idx.numel(), device=dev)
    I = K.indices()
    keep = free[I[0]] & free[I[1]]
    Kf = torch.sparse_coo_tensor(torch.stack([pos[I[0][keep]], pos[I[1][keep]]]), K.values()[keep],
                                 (idx.numel(), idx.numel())).coalesce()
    ff = f[idx]
    print(f"config 5 d={d}: {2 * nn} dofs, {idx.numel()} free, assembled in {time.perf_counter() - t0:.1f}s",
          flush=True)
    uf, true_res = cg(Kf, ff)
    u = torch.zeros(2 * nn, dtype=torch.float64, device=dev)
    u[idx] = uf
    u = u.cpu().numpy()
    n = 1 << d
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    z = O.z_index(ii, jj, d)
    qp = 4
    flat = np.zeros(2 * qp * 4**d)
    for m in range(3):
        for c in range(2):
            flat[z + 4**d * (m + qp * c)] = u[2 * ids[m] + c]
    if check:
        ref = np.load(os.path.join(HERE, f"conforming_c5_d{d}.npz"))
        uref = O.full([ref[f"cores_{k}"] for k in range(len(ref["ranks"]) - 1)])
        print(f"  vs reference splu fixture: rel diff {np.linalg.norm(flat - uref) / np.linalg.norm(uref):.2e}",
              flush=True)
        return
    cores = O.decompose_vector(flat, 1e-12)
    back = O.full(cores) if d <= 10 else None
    cerr = float(np.linalg.norm(back - flat) / np.linalg.norm(flat)) if back is not None else -1.0
    rng = np.random.default_rng(7)
    sidx = np.sort(rng.choice(flat.size, 256, replace=False))
    out = {f"cores_{k}": c for k, c in enumerate(cores)}
    out.update(ranks=np.asarray(O.ranks(cores), dtype=np.int64), norm=np.array(np.linalg.norm(flat)),
               compress_err=np.array(cerr), sample_idx=sidx.astype(np.int64), sample_val=flat[sidx],
               splu_residual=np.array(true_res), n_free=np.array(int(idx.numel())), d=np.array(d))
    os.makedirs("gpurun_out", exist_ok=True)
    path = os.path.join("gpurun_out", f"conforming_c5_d{d}.npz")
    np.savez_compressed(path, **out)
    print(f"  -> {path}: ranks max {max(O.ranks(cores))}, compress err {cerr:.2e}", flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]), "--check" in sys.argv)
