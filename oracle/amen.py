"""Numpy restatement of the reference AMEn-style solver (oracle; test
infrastructure).  Follows /root/reference/pkg/src/qttfem/solver.py:239-426
step for step with the direct local solver (``local_solver="direct"``, the
only setting that converges on the BASELINE problems).
TT objects are lists of numpy cores (oracle.tt conventions).
"""

from __future__ import annotations

import time

import numpy as np

from . import tt as O

DENSE_RESIDUAL_BITS = 22  # solver.py:24


def residual(K, u, f, dense_bits=DENSE_RESIDUAL_BITS):
    """solver.py:81-103 (TT path: norm after orthogonalisation, not Gram)."""
    fn = O.norm(f)
    if fn == 0.0:
        return 0.0
    if len(u) <= dense_bits:
        fd = O.full(f)
        return float(np.linalg.norm(O.apply_dense(K, O.full(u)) - fd) / np.linalg.norm(fd))
    y = O.add(O.matvec(K, u), O.scale(f, -1.0))
    return _orth_norm(y) / fn


def _orth_norm(cores):
    cs = [np.array(c) for c in cores]
    for k in range(len(cs) - 1, 0, -1):
        r, n, r2 = cs[k].shape
        q, rr = np.linalg.qr(cs[k].reshape(r, n * r2).T)
        cs[k - 1] = np.tensordot(cs[k - 1], rr.T, axes=(2, 0))
    return float(np.linalg.norm(cs[0]))


def _phi_l(phi, xr, a, xc):
    t = np.tensordot(phi, xr, axes=(0, 0))            # (a, y, i, X)
    t = np.tensordot(t, a, axes=([0, 2], [0, 1]))      # (y, X, j, b)
    return np.tensordot(t, xc, axes=([0, 2], [0, 1])).transpose(0, 1, 2)  # (X, b, Y)


def _phi_r(phi, xr, a, xc):
    t = np.tensordot(xr, phi, axes=(2, 0))             # (x, i, b, Y)
    t = np.tensordot(t, a, axes=([1, 2], [1, 3]))      # (x, Y, a, j)
    return np.tensordot(t, xc, axes=([1, 3], [2, 1]))  # (x, a, y)


def _psi_l(psi, xr, f):
    t = np.tensordot(psi, xr, axes=(0, 0))             # (q, i, X)
    return np.tensordot(t, f, axes=([0, 1], [0, 1]))   # (X, p)


def _psi_r(psi, xr, f):
    t = np.tensordot(xr, psi, axes=(2, 0))             # (x, i, p)
    return np.tensordot(t, f, axes=([1, 2], [1, 2]))   # (x, q)


def _rhs(psl, f, psr):
    return np.tensordot(np.tensordot(psl, f, axes=(1, 0)), psr, axes=(2, 1))  # (x, i, g)


def _dense(phl, a, phr):
    t = np.tensordot(phl, a, axes=(1, 0))              # (x, y, i, j, b)
    m = np.tensordot(t, phr, axes=(4, 1))              # (x, y, i, j, g, h)
    m = m.transpose(0, 2, 4, 1, 3, 5)
    n = phl.shape[0] * a.shape[1] * phr.shape[0]
    return m.reshape(n, n)


def _solve(phl, a, phr, rhs):
    mat = _dense(phl, a, phr)
    try:
        sol = np.linalg.solve(mat, rhs.reshape(-1))
    except np.linalg.LinAlgError:
        sol = np.linalg.lstsq(mat, rhs.reshape(-1), rcond=None)[0]
    return sol.reshape(rhs.shape)


def _proj(zl, xk, a, zr):
    t = np.tensordot(zl, xk, axes=(2, 0))              # (z, a, j, R)
    t = np.tensordot(t, a, axes=([1, 2], [0, 2]))      # (z, R, i, b)
    return np.tensordot(t, zr, axes=([3, 1], [1, 2]))  # (z, i, Z)


def _qr_left(core):
    r0, n, r1 = core.shape
    q, r = np.linalg.qr(core.reshape(r0 * n, r1))
    return q.reshape(r0, n, q.shape[1]), r


def _qr_right(core):
    r0, n, r1 = core.shape
    q, r = np.linalg.qr(core.reshape(r0, n * r1).T)
    return q.T.reshape(q.shape[1], n, r1), r.T


def _split_right(core, delta, rmax):
    r0, n, r1 = core.shape
    u, s, vt = np.linalg.svd(core.reshape(r0, n * r1), full_matrices=False)
    r = O.chop_nofloor(s, delta, rmax)
    return vt[:r].reshape(r, n, r1), u[:, :r] * s[:r]


def _init(rng, sizes, rank):
    d = len(sizes)
    rk = [1] + [rank] * (d - 1) + [1]
    cs = [rng.standard_normal((rk[k], sizes[k], rk[k + 1])) for k in range(d)]
    for k in range(d - 1, 0, -1):
        cs[k], c = _qr_right(cs[k])
        cs[k - 1] = np.tensordot(cs[k - 1], c, axes=(2, 0))
    return cs


def solve(K, f, eps=1e-8, max_sweeps=40, rho=4, seed=0, trunc_factor=0.5, max_rank=400,
          dense_bits=DENSE_RESIDUAL_BITS):
    """Returns dict(u, residual, sweeps, rank_history, residual_history, wall_time, converged)."""
    t0 = time.perf_counter()
    d = len(f)
    if O.norm(f) == 0.0:
        return dict(u=[np.zeros((1, c.shape[1], 1)) for c in f], residual=0.0, sweeps=0,
                    rank_history=(1,), residual_history=(0.0,), wall_time=0.0, converged=True)
    sizes = [c.shape[1] for c in f]
    rng = np.random.default_rng(seed)
    x = _init(rng, sizes, 2)
    z = _init(rng, sizes, rho)
    one3, one2 = np.ones((1, 1, 1)), np.ones((1, 1))
    phr, psr, zar, zfr = [None] * (d + 1), [None] * (d + 1), [None] * (d + 1), [None] * (d + 1)
    phr[d], psr[d], zar[d], zfr[d] = one3, one2, one3, one2
    for k in range(d - 1, -1, -1):
        phr[k] = _phi_r(phr[k + 1], x[k], K[k], x[k])
        psr[k] = _psi_r(psr[k + 1], x[k], f[k])
        zar[k] = _phi_r(zar[k + 1], z[k], K[k], x[k])
        zfr[k] = _psi_r(zfr[k + 1], z[k], f[k])
    phl, psl, zal, zfl = [None] * (d + 1), [None] * (d + 1), [None] * (d + 1), [None] * (d + 1)
    phl[0], psl[0], zal[0], zfl[0] = one3, one2, one3, one2
    ranks, hist = [], []
    res, res_prev, adapt, done = np.inf, np.inf, 1.0, 0
    for sweep in range(max_sweeps):
        for k in range(d):
            xk = _solve(phl[k], K[k], phr[k + 1], _rhs(psl[k], f[k], psr[k + 1]))
            x[k] = xk
            if k < d - 1:
                zloc = _rhs(zfl[k], f[k], zfr[k + 1]) - _proj(zal[k], xk, K[k], zar[k + 1])
                if np.linalg.norm(zloc) == 0.0:
                    zloc = rng.standard_normal(zloc.shape) * 1e-30
                z[k], _ = _qr_left(zloc)
                w = _rhs(psl[k], f[k], zfr[k + 1]) - _proj(phl[k], xk, K[k], zar[k + 1])
                xe = np.concatenate([x[k], w], axis=2)
                nxt = np.concatenate([x[k + 1], np.zeros((w.shape[2],) + x[k + 1].shape[1:])], axis=0)
                x[k], carry = _qr_left(xe)
                x[k + 1] = np.tensordot(carry, nxt, axes=(1, 0))
                phl[k + 1] = _phi_l(phl[k], x[k], K[k], x[k])
                psl[k + 1] = _psi_l(psl[k], x[k], f[k])
                zal[k + 1] = _phi_l(zal[k], z[k], K[k], x[k])
                zfl[k + 1] = _psi_l(zfl[k], z[k], f[k])
        delta = trunc_factor * eps * adapt * max(np.linalg.norm(x[d - 1]), 1e-300) / np.sqrt(d)
        for k in range(d - 1, -1, -1):
            xk = _solve(phl[k], K[k], phr[k + 1], _rhs(psl[k], f[k], psr[k + 1]))
            if k > 0:
                x[k], carry = _split_right(xk, delta, max_rank)
                x[k - 1] = np.tensordot(x[k - 1], carry, axes=(2, 0))
                phr[k] = _phi_r(phr[k + 1], x[k], K[k], x[k])
                psr[k] = _psi_r(psr[k + 1], x[k], f[k])
                zk = z[k] if np.linalg.norm(z[k]) != 0.0 else rng.standard_normal(z[k].shape) * 1e-30
                z[k], _ = _qr_right(zk)
                zar[k] = _phi_r(zar[k + 1], z[k], K[k], x[k])
                zfr[k] = _psi_r(zfr[k + 1], z[k], f[k])
            else:
                x[k] = xk
        done = sweep + 1
        ranks.append(max(c.shape[0] for c in x[1:]) if d > 1 else 1)
        res = residual(K, x, f, dense_bits)
        hist.append(res)
        if res <= eps:
            break
        if res > 0.7 * res_prev and adapt > 2.0**-44:
            adapt *= 0.25
        res_prev = res
    u = [c.copy() for c in x]
    if res <= eps:
        for fac in (0.5, 0.25, 0.1, 0.03, 0.01, 0.003):
            cand = O.round_tt(u, fac * eps)
            r = residual(K, cand, f, dense_bits)
            if r <= eps:
                u, res = cand, r
                break
    return dict(u=u, residual=float(res), sweeps=done, rank_history=tuple(ranks),
                residual_history=tuple(hist), wall_time=time.perf_counter() - t0,
                converged=bool(res <= eps))
