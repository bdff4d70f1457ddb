"""Numpy restatement of the reference TT algebra (oracle; test infrastructure).

A TT vector is a python list of float64 cores shaped ``(r_prev, n, r_next)``;
a TT matrix is a list of cores ``(r_prev, n_row, n_col, r_next)``.  The flat
index is LSB-first (core l carries bit l-1), see
/root/reference/pkg/src/qttfem/ttcore.py:3-10.

Every routine names the reference lines it restates.  Nothing in here is
used by the product; see ``oracle/__init__.py``.
"""

from __future__ import annotations

import numpy as np

EPS64 = float(np.finfo(np.float64).eps)
DENSE_GUARD_BITS = 24  # ttcore.py:46


# ------------------------------------------------------------------ helpers


def is_matrix(cores) -> bool:
    return cores[0].ndim == 4


def merge(cores):
    """Order-3 views; matrix mode k = i + n*j (ttcore.py:159-167)."""
    if not is_matrix(cores):
        return [np.asarray(c, dtype=np.float64) for c in cores]
    out = []
    for c in cores:
        r0, n, m, r1 = c.shape
        out.append(np.ascontiguousarray(np.swapaxes(c, 1, 2)).reshape(r0, n * m, r1))
    return out


def unmerge(merged, rows, cols):
    """Inverse of :func:`merge` (ttcore.py:170-172)."""
    out = []
    for c, n, m in zip(merged, rows, cols):
        r0, _, r1 = c.shape
        out.append(np.ascontiguousarray(np.swapaxes(c.reshape(r0, m, n, r1), 1, 2)))
    return out


def ranks(cores):
    return (1,) + tuple(int(c.shape[-1]) for c in cores)


# ------------------------------------------------------------ truncation


def chop(s, delta: float) -> int:
    """Rank kept by the reference rule (ttcore.py:175-190).

    Keep the smallest r whose discarded tail energy sqrt(sum s[r:]^2) is
    <= max(delta, s0 * max(len, 2) * eps); at least 1.
    """
    s = np.asarray(s, dtype=np.float64)
    if s.size == 0:
        return 1
    thr = max(float(delta), float(s[0] * max(s.size, 2) * EPS64))
    tails = np.sqrt(np.cumsum(s[::-1] ** 2))[::-1]  # tails[k] = ||s[k:]||
    above = np.nonzero(tails > thr)[0]
    return int(above[-1] + 1) if above.size else 1


def chop_nofloor(s, delta: float, rmax: int) -> int:
    """Solver truncation rule without the eps floor (solver.py:221-236)."""
    s = np.asarray(s, dtype=np.float64)
    tails = np.sqrt(np.cumsum(s[::-1] ** 2))[::-1]
    above = np.nonzero(tails > delta)[0]
    r = int(above[-1] + 1) if above.size else 1
    return max(1, min(r, rmax))


# --------------------------------------------------------------- TT-SVD


def _sweep_svd(tensor, sizes, delta):
    """Sequential truncated-SVD sweep (ttcore.py:193-208)."""
    cores = []
    rest = tensor
    rp = 1
    for n in sizes[:-1]:
        mat = rest.reshape(rp * n, -1)
        u, s, vt = np.linalg.svd(mat, full_matrices=False)
        r = chop(s, delta)
        cores.append(u[:, :r].reshape(rp, n, r))
        rest = s[:r, None] * vt[:r]
        rp = r
    cores.append(rest.reshape(rp, sizes[-1], 1))
    return cores


def decompose_vector(v, eps: float, sizes=None):
    """tt_decompose for a 1-D array (ttcore.py:211-235)."""
    v = np.asarray(v, dtype=np.float64).ravel()
    if sizes is None:
        d = v.size.bit_length() - 1
        sizes = (2,) * d
    sizes = tuple(int(x) for x in sizes)
    nrm = float(np.linalg.norm(v))
    if nrm == 0.0:
        return [np.zeros((1, n, 1)) for n in sizes]
    delta = eps / np.sqrt(max(len(sizes) - 1, 1)) * nrm
    return _sweep_svd(v.reshape(sizes, order="F"), sizes, delta)


def decompose_matrix(a, eps: float, rows=None, cols=None):
    """tt_decompose for a square 2-D array (ttcore.py:236-263)."""
    a = np.asarray(a, dtype=np.float64)
    if rows is None:
        d = a.shape[0].bit_length() - 1
        rows = cols = (2,) * d
    d = len(rows)
    delta = eps / np.sqrt(max(d - 1, 1)) * float(np.linalg.norm(a))
    t = a.reshape(tuple(rows) + tuple(cols), order="F")
    perm = [ax for l in range(d) for ax in (l, d + l)]
    merged_sizes = [rows[l] * cols[l] for l in range(d)]
    t = t.transpose(perm).reshape(merged_sizes, order="F")
    return unmerge(_sweep_svd(t, merged_sizes, delta), rows, cols)


# --------------------------------------------------------------- dense


def full(cores):
    """Dense realisation (ttcore.py:267-293)."""
    if not is_matrix(cores):
        acc = np.ones((1, 1))
        for c in cores:
            acc = np.tensordot(acc, c, axes=(-1, 0))
        return acc.reshape(-1, order="C").reshape(
            tuple(c.shape[1] for c in cores), order="C"
        ).ravel(order="F")
    rows = [c.shape[1] for c in cores]
    cols = [c.shape[2] for c in cores]
    acc = np.ones((1, 1))
    for c in merge(cores):
        acc = np.tensordot(acc, c, axes=(-1, 0))
    acc = acc.reshape(acc.shape[1:-1])
    split = [x for l in range(len(cores)) for x in (rows[l], cols[l])]
    acc = acc.reshape(split, order="F")
    d = len(cores)
    acc = acc.transpose(list(range(0, 2 * d, 2)) + list(range(1, 2 * d, 2)))
    return acc.reshape(int(np.prod(rows)), int(np.prod(cols)), order="F")


# ------------------------------------------------------------- rounding


def _qr_sweep_right(cores):
    """Right-to-left orthogonalisation (ttcore.py:296-306)."""
    cores = [np.array(c, dtype=np.float64) for c in cores]
    for k in range(len(cores) - 1, 0, -1):
        r, n, r2 = cores[k].shape
        q, rr = np.linalg.qr(cores[k].reshape(r, n * r2).T)
        cores[k] = np.ascontiguousarray(q.T).reshape(q.shape[1], n, r2)
        cores[k - 1] = np.tensordot(cores[k - 1], rr.T, axes=(2, 0))
    return cores


def _svd_sweep_left(cores, delta):
    """Left-to-right truncated SVD sweep (ttcore.py:309-319)."""
    for k in range(len(cores) - 1):
        r, n, r2 = cores[k].shape
        u, s, vt = np.linalg.svd(cores[k].reshape(r * n, r2), full_matrices=False)
        keep = min(chop(s, delta), cores[k + 1].shape[0])
        cores[k] = u[:, :keep].reshape(r, n, keep)
        cores[k + 1] = np.tensordot(s[:keep, None] * vt[:keep], cores[k + 1], axes=(1, 0))
    return cores


def gram_norm(merged) -> float:
    """Norm by Gram accumulation (ttcore.py:341-347)."""
    g = np.ones((1, 1))
    for c in merged:
        half = np.tensordot(g, c, axes=(1, 0))  # (a, n, d)
        g = np.tensordot(c, half, axes=([0, 1], [0, 1]))
    return float(np.sqrt(max(g[0, 0], 0.0)))


def round_tt(cores, eps: float):
    """tt_round (ttcore.py:322-338)."""
    mat = is_matrix(cores)
    m = merge(cores)
    d = len(m)
    delta = eps / np.sqrt(max(d - 1, 1)) * gram_norm(m)
    out = _svd_sweep_left(_qr_sweep_right(m), delta)
    if mat:
        return unmerge(out, [c.shape[1] for c in cores], [c.shape[2] for c in cores])
    return out


def norm(cores) -> float:
    return gram_norm(merge(cores))


def dot(a, b) -> float:
    """tt_dot (ttcore.py:355-363)."""
    g = np.ones((1, 1))
    for ca, cb in zip(a, b):
        half = np.tensordot(g, cb, axes=(1, 0))
        g = np.tensordot(ca, half, axes=([0, 1], [0, 1]))
    return float(g[0, 0])


# ----------------------------------------------------- structural algebra


def add(a, b):
    """Block-diagonal rank concatenation (ttcore.py:380-411)."""
    mat = is_matrix(a)
    ma, mb = merge(a), merge(b)
    d = len(ma)
    out = []
    for k, (x, y) in enumerate(zip(ma, mb)):
        if d == 1:
            out.append(x + y)
            continue
        first, last = k == 0, k == d - 1
        r0 = 1 if first else x.shape[0] + y.shape[0]
        r1 = 1 if last else x.shape[2] + y.shape[2]
        c = np.zeros((r0, x.shape[1], r1))
        o0 = 0 if first else x.shape[0]
        o1 = 0 if last else x.shape[2]
        c[: x.shape[0], :, : x.shape[2]] = x
        c[o0 : o0 + y.shape[0], :, o1 : o1 + y.shape[2]] = y
        out.append(c)
    if mat:
        return unmerge(out, [c.shape[1] for c in a], [c.shape[2] for c in a])
    return out


def scale(a, s):
    """Scale the first core (ttcore.py:414-418)."""
    out = [np.array(c, dtype=np.float64) for c in a]
    out[0] = out[0] * float(s)
    return out


def hadamard(a, b):
    """Elementwise product, ranks multiply (ttcore.py:421-440)."""
    mat = is_matrix(a)
    out = []
    for x, y in zip(merge(a), merge(b)):
        c = np.einsum("anb,cnd->acnbd", x, y)
        out.append(c.reshape(x.shape[0] * y.shape[0], x.shape[1], x.shape[2] * y.shape[2]))
    if mat:
        return unmerge(out, [c.shape[1] for c in a], [c.shape[2] for c in a])
    return out


def matvec(A, x):
    """Exact core-wise product, A-rank slow (ttcore.py:443-455)."""
    out = []
    for a, v in zip(A, x):
        c = np.einsum("pijq,sjt->psiqt", a, v)
        out.append(c.reshape(a.shape[0] * v.shape[0], a.shape[1], a.shape[3] * v.shape[2]))
    return out


def matmat(A, B):
    """Exact core-wise product (ttcore.py:458-470)."""
    out = []
    for a, b in zip(A, B):
        c = np.einsum("pijq,sjkt->psikqt", a, b)
        out.append(
            c.reshape(a.shape[0] * b.shape[0], a.shape[1], b.shape[2], a.shape[3] * b.shape[3])
        )
    return out


def transpose(A):
    return [np.ascontiguousarray(np.swapaxes(c, 1, 2)) for c in A]


def diag(v):
    """Diagonal operator (ttcore.py:478-486)."""
    out = []
    for c in v:
        r0, n, r1 = c.shape
        m = np.zeros((r0, n, n, r1))
        for i in range(n):
            m[:, i, i, :] = c[:, i, :]
        out.append(m)
    return out


def kron(A, B):
    """B's cores first (ttcore.py:489-498)."""
    return [np.array(c) for c in B] + [np.array(c) for c in A]


def zkron(A, B):
    """Bit-interleaved Kronecker product (ttcore.py:501-539)."""
    mat = is_matrix(A)
    ma, mb = merge(A), merge(B)
    out, rows, cols = [], [], []
    for k in range(len(ma)):
        a, b = ma[k], mb[k]
        ra0, na, ra1 = a.shape
        rb0, nb, rb1 = b.shape
        fast = np.einsum("bnc,ad->bancd", b, np.eye(ra0)).reshape(rb0 * ra0, nb, rb1 * ra0)
        slow = np.einsum("anb,cd->candb", a, np.eye(rb1)).reshape(rb1 * ra0, na, rb1 * ra1)
        out += [fast, slow]
        if mat:
            rows += [B[k].shape[1], A[k].shape[1]]
            cols += [B[k].shape[2], A[k].shape[2]]
    return unmerge(out, rows, cols) if mat else out


def ones(sizes):
    return [np.ones((1, n, 1)) for n in sizes]


def identity(sizes):
    return [np.eye(n).reshape(1, n, n, 1) for n in sizes]


def slice_mode(cores, mode, index):
    """Fix one mode and absorb it into a neighbour (ttcore.py:566-586)."""
    cs = [np.array(c) for c in cores]
    sl = cs[mode][:, index, :]
    del cs[mode]
    if mode == 0:
        cs[0] = np.einsum("ab,bnc->anc", sl, cs[0])
    else:
        cs[mode - 1] = np.einsum("anb,bc->anc", cs[mode - 1], sl)
    return cs


def apply_dense(A, v):
    """Dense vector times TT operator, core by core (solver.py:57-73)."""
    cols = [c.shape[2] for c in A]
    t = np.asarray(v, dtype=np.float64).reshape((1,) + tuple(cols), order="F")
    for c in A:
        # t: (bond, col_k, rest..., rows_done...)
        t = np.tensordot(c, t, axes=([0, 2], [0, 1]))  # (row_k, bond', rest..., done...)
        t = np.moveaxis(t, 0, -1)
    return t.reshape(-1, order="F")


# ------------------------------------------------------------ index maps


def spread_bits(x, d):
    x = np.asarray(x, dtype=np.int64)
    z = np.zeros_like(x)
    for b in range(d):
        z |= ((x >> b) & 1) << (2 * b)
    return z


def z_index(i, j, d):
    """indexing.py:58-64"""
    return spread_bits(i, d) | (spread_bits(j, d) << 1)


def zorder_permutation(d):
    """perm[Z(i,j)] = i + 2^d j (indexing.py:87-99)."""
    n = 1 << d
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    perm = np.empty(n * n, dtype=np.int64)
    perm[z_index(ii, jj, d).ravel()] = (ii + n * jj).ravel()
    return perm


def zorder_dof_permutation(d):
    """Entry 2Z+c maps to 2L+c (indexing.py:102-112)."""
    p = zorder_permutation(d)
    out = np.empty(2 * p.size, dtype=np.int64)
    out[0::2] = 2 * p
    out[1::2] = 2 * p + 1
    return out
