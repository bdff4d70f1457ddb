"""AMEn-style TT solve of K u = f on the device: drop-in for ``qttfem.solver``
(solver.py:21-426).

Same algorithm and control flow as the reference: one-site ALS sweeps with
residual-projection enrichment by a rank-``enrichment_rank`` companion
(forward half-sweep), SVD truncation at
delta = trunc_factor * eps * adapt * ||x_d|| / sqrt(d) (backward half-sweep),
relative residual after every sweep, stall adaptation, final compression.
Every contraction runs on the DMMA GEMM of libqttb200.so, local systems are
solved by the device LU (``qtt_dense_solve``), QR/SVD by the device
Householder / Jacobi kernels.  The only data that reaches the host per sweep
are the scalars that steer control flow (residual, truncation ranks).

Initial cores come from numpy ``default_rng(seed)`` exactly as in the
reference (solver.py:258-261, 419-426) and are uploaded.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._dense import dense_solve_colmajor, mm, qr_colmajor, svd_left_colmajor
from .ttcore import (
    TTMatrix,
    TTVector,
    _concat,
    tt_add,
    tt_contract_device,
    tt_decompose,
    tt_matvec,
    tt_norm,
    tt_round,
    tt_sub,
)

__all__ = ["SolverConfig", "SolveOutcome", "solve", "residual", "apply_tt_matrix"]

_RELEASE_DIM = 30000  # local systems above ~7 GB trim the allocator caches first
_DENSE_LOCAL_LIMIT = 1200  # kept for API parity (solver.py:23); local solves are direct

_TRACE = bool(__import__("os").environ.get("QTT_AMEN_TRACE"))

# Optional phase timing (synchronising; diagnostics only): set PROFILE = {}.
PROFILE = None


class _phase:
    def __init__(self, name):
        self.name = name

    def __enter__(self):
        if PROFILE is not None:
            torch.cuda.synchronize()
            self.t = time.perf_counter()

    def __exit__(self, *exc):
        if PROFILE is not None:
            torch.cuda.synchronize()
            PROFILE[self.name] = PROFILE.get(self.name, 0.0) + time.perf_counter() - self.t
_DENSE_RESIDUAL_BITS = 22  # materialise vectors up to 2^22 entries (solver.py:24)


@dataclass(frozen=True)
class SolverConfig:
    epsilon: float = 1e-8
    max_sweeps: int = 40
    enrichment_rank: int = 4
    # direct: dense device LU for every local system; iterative/auto: device
    # GMRES (warm start, restart 40, reference tolerance) above
    # _ITERATIVE_MIN_DIM unknowns, dense LU below and as fallback
    local_solver: str = "auto"
    seed: int = 0
    trunc_factor: float = 0.5
    max_rank: int = 400
    # "reference": SVD truncation at delta with the stall adaptation of
    # solver.py:374-380 (drop-in behaviour).  "residual": the AMEn
    # local-residual rule (Dolgov & Savostyanov 2014): keep the smallest rank
    # whose truncated local solution still satisfies the local system to
    # trunc_factor * epsilon / sqrt(d) (no stall adaptation needed).
    truncation: str = "reference"
    # Extension (0 = reference rule): with the residual truncation rule, the
    # local tolerance is relaxed to local_rtol_factor * (latest known global
    # residual) while that exceeds the reference's 0.02 * epsilon, i.e.
    # inexact local solves in the early sweeps (no accuracy is lost at
    # convergence: the bound tightens with the residual).  Sweep s uses the
    # residual of sweep s-2 on every path (the residual of sweep s-1 may
    # still be in flight on the side stream when sweep s starts).
    local_rtol_factor: float = 0.0
    # Extension (0 = reference behaviour: run until residual <= epsilon or
    # max_sweeps): stop once the residual has not improved on its best value
    # by 2x for stall_sweeps consecutive sweeps and return the best iterate.
    # For operators whose attainable FP64 residual ~ eps_mach * ||K|| ||u|| /
    # ||f|| exceeds epsilon (config 5 at d >= 8) the sweeps
    # past that floor only re-shuffle rounding noise.  ``converged`` still
    # reports residual <= epsilon.
    stall_sweeps: int = 0
    # Extension (0 = reference behaviour): iterative refinement after the
    # sweeps when the residual is still above epsilon.  Each step forms the
    # dense residual r = f - K u on the device, compresses it by TT-SVD,
    # solves K e = r with the same AMEn to the loose relative tolerance
    # refine_tol and keeps u + e if its residual is smaller.  All floors of a
    # sweep (truncation relative to ||u||, local tolerances relative to the
    # local right-hand side) scale with ||r|| instead of ||f|| in the
    # correction solve, which is what lets the penalty-coupled systems of
    # config 5 past the residual their sweeps stall at.
    refine_steps: int = 0
    refine_tol: float = 1e-3

    def __post_init__(self):
        if self.epsilon <= 0:
            raise ValueError("epsilon must be positive")
        if self.max_sweeps < 1:
            raise ValueError("max_sweeps must be >= 1")
        if self.local_solver not in ("auto", "direct", "iterative"):
            raise ValueError(f"unknown local solver {self.local_solver!r}")
        if self.truncation not in ("reference", "residual"):
            raise ValueError(f"unknown truncation rule {self.truncation!r}")
        if self.stall_sweeps < 0:
            raise ValueError("stall_sweeps must be >= 0")
        if self.refine_steps < 0 or not self.refine_tol > 0:
            raise ValueError("refine_steps must be >= 0 and refine_tol positive")


@dataclass(frozen=True)
class SolveOutcome:
    u: TTVector
    residual: float
    sweeps: int
    rank_history: tuple
    residual_history: tuple
    wall_time: float
    converged: bool


# ------------------------------------------------------------- residual


def apply_tt_matrix(A: TTMatrix, v):
    """Dense matvec of a TT operator on the device (solver.py:57-73).  A host
    array comes back as a host numpy array, as in the reference; a torch
    tensor stays on the device."""
    dev = _lib.device()
    on_host = not isinstance(v, torch.Tensor)
    x = v if not on_host else torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
    x = x.to(device=dev, dtype=torch.float64).contiguous()
    out = torch.empty(A.shape[0], dtype=torch.float64, device=dev)
    lay = A._layout()
    _lib.call("qtt_dense_apply", ctypes.byref(lay), _lib.ptr(A.data), _lib.ptr(x), _lib.ptr(out),
              _lib.stream_handle())
    return out.cpu().numpy() if on_host else out


def _apply_tt_to_tt(K: TTMatrix, u: TTVector) -> torch.Tensor:
    """Dense y = K u for a TT operator and a TT vector (the dense residual
    path of solver.py:81-103) without materialising u: the left half of the
    cores is contracted into L[i_low, a, b] (operator rank a, vector rank b),
    the right half into R[a, b, i_high], and y = L R is one GEMM.  Flops
    ~ 2^(D/2) r_K r_u (r_K + r_u) per core plus 2^D r_K r_u, against
    ~ 2^D r_K^2 per core for the dense chain over a materialised u (about 5x
    fewer at the config-4 ranks).  Returns the flat (row-index) vector."""
    Kc, uc = K.device_cores, u.device_cores
    D = len(uc)
    m = D // 2
    dev = u.data.device
    L = torch.ones((1, 1, 1), dtype=torch.float64, device=dev)
    for l in range(m):
        rk, ni, nj, rk2 = Kc[l].shape
        ru, _, ru2 = uc[l].shape
        P = L.shape[0]
        T = mm(L.reshape(P * rk, ru), uc[l].reshape(ru, nj * ru2))  # (P, a, j, b')
        T = T.view(P, rk, nj, ru2).permute(0, 3, 1, 2).reshape(P * ru2, rk * nj)
        Kp = Kc[l].permute(0, 2, 1, 3).reshape(rk * nj, ni * rk2)  # ((a, j), (i, a'))
        U = mm(T, Kp).view(P, ru2, ni, rk2)
        L = U.permute(2, 0, 3, 1).reshape(ni * P, rk2, ru2)  # new bit is the slowest
    R = torch.ones((1, 1, 1), dtype=torch.float64, device=dev)
    for l in range(D - 1, m - 1, -1):
        rk, ni, nj, rk2 = Kc[l].shape
        ru, _, ru2 = uc[l].shape
        Q = R.shape[2]
        T = mm(uc[l].reshape(ru * nj, ru2), R.permute(1, 0, 2).reshape(ru2, rk2 * Q))  # (b, j, a', Q)
        T = T.view(ru, nj, rk2, Q).permute(0, 3, 1, 2).reshape(ru * Q, nj * rk2)
        Kp = Kc[l].permute(2, 3, 0, 1).reshape(nj * rk2, rk * ni)  # ((j, a'), (a, i))
        U = mm(T, Kp).view(ru, Q, rk, ni)
        R = U.permute(2, 0, 1, 3).reshape(rk, ru, Q * ni)  # new bit is the fastest
    P, Q = L.shape[0], R.shape[2]
    # y[i_low + P i_high] = sum_ab L[i_low, a, b] R[a, b, i_high]
    return mm(R.reshape(-1, Q), L.reshape(P, -1), ta=True, tb=True).view(-1)


def residual(K: TTMatrix, u: TTVector, f: TTVector, rounding_eps=None) -> float:
    """||K u - f|| / ||f|| (solver.py:81-103).  Dense on the device up to
    2^_DENSE_RESIDUAL_BITS entries, else in TT arithmetic with the norm taken
    after orthogonalisation (no sqrt(eps) floor)."""
    fn = tt_norm(f)
    if fn == 0.0:
        return 0.0
    if len(u.device_cores) <= _DENSE_RESIDUAL_BITS:
        fd = tt_contract_device(f)
        r = _apply_tt_to_tt(K, u) - fd
        return float(torch.linalg.vector_norm(r) / torch.linalg.vector_norm(fd))
    y = tt_sub(tt_matvec(K, u), f)
    if rounding_eps is not None:
        y = tt_round(y, rounding_eps / 100.0)
    return tt_norm(y) / fn


_SIDE = {}


class _AsyncResidual:
    """residual(K, u, f) on the dense path, enqueued on a side stream
    (same operations and order, so the same value); value() waits."""

    def __init__(self, K: TTMatrix, u: TTVector, fd: torch.Tensor):
        dev = torch.cuda.current_device()
        side = _SIDE.get(dev)
        if side is None:
            side = _SIDE[dev] = torch.cuda.Stream(device=dev)
        main = torch.cuda.current_stream()
        side.wait_stream(main)
        u.data.record_stream(side)
        fd.record_stream(side)
        K.data.record_stream(side)
        with torch.cuda.stream(side):
            r = _apply_tt_to_tt(K, u) - fd
            self._val = torch.linalg.vector_norm(r) / torch.linalg.vector_norm(fd)
            self._ev = torch.cuda.Event()
            self._ev.record(side)

    def ready(self) -> bool:
        return self._ev.query()

    def value(self) -> float:
        self._ev.synchronize()
        return float(self._val)


# ------------------------------------------------- interface contractions


def _phi_left(phi, xrow, a_p, xcol):
    """(x,a,y),(x,i,X),A,(y,j,Y) -> (X,b,Y)   (solver.py:109-112)."""
    x, a, y = phi.shape
    _, n, X = xrow.shape
    Y = xcol.shape[2]
    b = a_p["rb"]
    t1 = mm(phi.reshape(x, a * y), xrow.reshape(x, n * X), ta=True)  # (a,y,i,X)
    t1 = t1.view(a, y, n, X).permute(1, 3, 0, 2).reshape(y * X, a * n)
    t2 = mm(t1, a_p["ai_jb"])  # (y,X,j,b)
    t2 = t2.view(y, X, n, b).permute(1, 3, 0, 2).reshape(X * b, y * n)
    return mm(t2, xcol.reshape(y * n, Y)).view(X, b, Y)


def _phi_right(phi, xrow, a_p, xcol):
    """(X,b,Y),(x,i,X),A,(y,j,Y) -> (x,a,y)   (solver.py:115-118)."""
    X, b, Y = phi.shape
    x, n, _ = xrow.shape
    y = xcol.shape[0]
    a = a_p["ra"]
    t1 = mm(xrow.reshape(x * n, X), phi.reshape(X, b * Y))  # (x,i,b,Y)
    t1 = t1.view(x, n, b, Y).permute(0, 3, 1, 2).reshape(x * Y, n * b)
    t2 = mm(t1, a_p["ib_aj"])  # (x,Y,a,j)
    t2 = t2.view(x, Y, a, n).permute(0, 2, 1, 3).reshape(x * a, Y * n)
    xc = xcol.permute(2, 1, 0).reshape(Y * n, y)
    return mm(t2, xc).view(x, a, y)


def _psi_left(psi, xrow, f):
    """(x,q),(x,i,X),(q,i,p) -> (X,p)   (solver.py:121-123)."""
    x, q = psi.shape
    _, n, X = xrow.shape
    t = mm(psi, xrow.reshape(x, n * X), ta=True)  # (q,i,X)
    return mm(t.view(q * n, X), f.reshape(q * n, f.shape[2]), ta=True)


def _psi_right(psi, xrow, f):
    """(X,p),(x,i,X),(q,i,p) -> (x,q)   (solver.py:126-128)."""
    x, n, X = xrow.shape
    t = mm(xrow.reshape(x * n, X), psi)  # (x,i,p)
    return mm(t.view(x, n * psi.shape[1]), f.reshape(f.shape[0], n * f.shape[2]), tb=True)


def _local_rhs(psi_l, f, psi_r):
    """(x,q),(q,i,p),(g,p) -> (x,i,g)   (solver.py:131-133)."""
    x, q = psi_l.shape
    _, n, p = f.shape
    t = mm(psi_l, f.reshape(q, n * p))
    return mm(t.view(x * n, p), psi_r, tb=True).view(x, n, psi_r.shape[0])


def _local_matrix_cm(phi_l, a_p, phi_r):
    """Column-major local operator M[(x,i,g),(y,j,h)] (solver.py:148-152):
    memory laid out as the C-order tensor (y,j,h,x,i,g)."""
    x, a, y = phi_l.shape
    g, b, h = phi_r.shape
    n = a_p["n"]
    pl = phi_l.permute(0, 2, 1).reshape(x * y, a)
    t = mm(pl, a_p["a_ijb"])  # (x,y,i,j,b)
    pr = phi_r.permute(1, 0, 2).reshape(b, g * h)
    mat = mm(t.view(x * y * n * n, b), pr)  # (x,y,i,j,g,h)
    mat = mat.view(x, y, n, n, g, h).permute(1, 3, 5, 0, 2, 4).contiguous()
    return mat.view(-1)


_LOCAL_HOOK = None  # diagnostics: called with (phi_l, a_p, phi_r, rhs, x_cur, sol)

# "auto"/"iterative": local systems above this dimension are solved by
# warm-started GMRES on the structured operator (no dense matrix); at and
# below it the dense device LU is cheaper than a few dozen GMRES iterations.
_ITERATIVE_MIN_DIM = 8192
_GMRES_RESTART = 40
_GMRES_MAXIT = 400
# beyond this dimension a dense fallback costs seconds ((2/3) N^3 flops: 0.4 s
# at 24,000, 6 s at 60,000, which is what a stalling config-5 sweep used to
# spend on local systems GMRES cannot resolve below the FP64 floor); the
# warm-started GMRES iterate, never worse than the current core, is kept
_DENSE_FALLBACK_MAX = 24000


def _local_matvec(phi_l, a_p, phi_r, x):
    """M x for the local operator M[(x,i,g),(y,j,h)] = sum_ab phi_l[x,a,y]
    A[a,i,j,b] phi_r[g,b,h] (solver.py:136-139): qtt_local_apply (three DMMA
    GEMMs and two permutations, one C-ABI call)."""
    rl, n, rr = x.shape
    y = torch.empty_like(x)
    _lib.call("qtt_local_apply", ctypes.c_int64(rl), ctypes.c_int64(n), ctypes.c_int64(rr),
              ctypes.c_int64(a_p["ra"]), ctypes.c_int64(a_p["rb"]), _lib.ptr(phi_l.contiguous()),
              _lib.ptr(a_p["aj_ib"]), _lib.ptr(phi_r.contiguous()), _lib.ptr(x.contiguous()),
              _lib.ptr(y), _lib.stream_handle())
    return y


def _gmres(phi_l, a_p, phi_r, b, x0, rtol, restart=_GMRES_RESTART, maxit=_GMRES_MAXIT,
           abort_early=False):
    """Restarted GMRES (solver.py:186-195 uses scipy's, restart 40) on the
    structured local operator: qtt_local_gmres runs the whole iteration on
    the device, driven from C++ (CGS2 Arnoldi, host Givens).  Returns
    (x, converged, iterations)."""
    rl, n, rr = b.shape
    x = x0.contiguous().clone()
    its = ctypes.c_int32(0)
    conv = ctypes.c_int32(0)
    _lib.call("qtt_local_gmres", ctypes.c_int64(rl), ctypes.c_int64(n), ctypes.c_int64(rr),
              ctypes.c_int64(a_p["ra"]), ctypes.c_int64(a_p["rb"]), _lib.ptr(phi_l.contiguous()),
              _lib.ptr(a_p["aj_ib"]), _lib.ptr(phi_r.contiguous()), _lib.ptr(b.contiguous()),
              _lib.ptr(x), _lib.ptr(x), ctypes.c_double(rtol), ctypes.c_int32(restart),
              ctypes.c_int32(maxit), ctypes.c_int32(1 if abort_early else 0), ctypes.byref(its),
              ctypes.byref(conv), _lib.stream_handle())
    return x, bool(conv.value), int(its.value)


def _solve_local(phi_l, a_p, phi_r, rhs, keep=False, x_cur=None, cfg=None, rtol=1e-12):
    """Local system M x = rhs (solver.py:162-196).  ``direct``: dense device
    LU (+ refinement / QR fallback).  ``iterative``/``auto`` above
    _ITERATIVE_MIN_DIM: GMRES warm-started from the current core, with the
    reference's local tolerance; a dense solve is the fallback when GMRES
    does not converge.  With ``keep`` also returns the dense operator (None
    on the iterative path)."""
    rl, n, rr = rhs.shape
    dim = rl * n * rr
    iterative = cfg is not None and cfg.local_solver != "direct" and dim > _ITERATIVE_MIN_DIM
    if iterative:
        x0 = x_cur if (x_cur is not None and tuple(x_cur.shape) == tuple(rhs.shape)) else torch.zeros_like(rhs)
        tg = PROFILE.get("local_gmres", 0.0) if PROFILE is not None else 0.0
        with _phase("local_gmres"):
            sol, ok, its = _gmres(phi_l, a_p, phi_r, rhs, x0, rtol, abort_early=dim <= _DENSE_FALLBACK_MAX)
        if PROFILE is not None:
            PROFILE["gmres_its"] = PROFILE.get("gmres_its", 0) + its
            PROFILE.setdefault("calls", []).append(
                ("gmres", rl, a_p["ra"], rr, its, bool(ok), round(PROFILE["local_gmres"] - tg, 4)))
        if ok or dim > _DENSE_FALLBACK_MAX:
            if _LOCAL_HOOK is not None:
                _LOCAL_HOOK(phi_l, a_p, phi_r, rhs, x_cur, sol)
            return (sol, None) if keep else sol
        if PROFILE is not None:
            PROFILE["gmres_fallbacks"] = PROFILE.get("gmres_fallbacks", 0) + 1
    if dim > _RELEASE_DIM:
        # local systems grow sweep by sweep; stale blocks of either cache
        # would otherwise pin tens of GB (see _lib.release_cached)
        _lib.release_cached()
    with _phase("local_matrix"):
        mcm = _local_matrix_cm(phi_l, a_p, phi_r)
    tl = PROFILE.get("local_lu", 0.0) if PROFILE is not None else 0.0
    with _phase("local_lu"):
        sol, _ = dense_solve_colmajor(mcm, dim, rhs.reshape(-1))
    if PROFILE is not None:
        PROFILE.setdefault("calls", []).append(
            ("lu", rl, a_p["ra"], rr, dim, True, round(PROFILE["local_lu"] - tl, 4)))
    if _LOCAL_HOOK is not None:
        _LOCAL_HOOK(phi_l, a_p, phi_r, rhs, x_cur, sol.view(rl, n, rr))
    if keep:
        return sol.view(rl, n, rr), mcm
    return sol.view(rl, n, rr)


def _proj_a(zl, xk, a_p, zr):
    """einsum zaL,LjR,aijb,ZbR -> ziZ (solver.py:306-313, 318-323)."""
    z, a, L = zl.shape
    _, n, R = xk.shape
    Z, b, _ = zr.shape
    t = mm(zl.reshape(z * a, L), xk.reshape(L, n * R))  # (z,a,j,R)
    t = t.view(z, a, n, R).permute(0, 3, 1, 2).reshape(z * R, a * n)
    t2 = mm(t, a_p["aj_ib"])  # (z,R,i,b)
    t2 = t2.view(z, R, n, b).permute(0, 2, 3, 1).reshape(z * n, b * R)
    return mm(t2, zr.reshape(Z, b * R), tb=True).view(z, n, Z)


# ---------------------------------------------------------- QR and SVD


def _qr_core_left(core):
    rl, n, rr = core.shape
    cm = core.reshape(rl * n, rr).t().contiguous()  # column-major (rl n x rr)
    q, r, k = qr_colmajor(cm, rl * n, rr)
    qc = q.view(k, rl * n).t().contiguous().view(rl, n, k)
    rc = r.view(rr, k).t().contiguous()  # (k, rr)
    return qc, rc


def _qr_core_right(core):
    rl, n, rr = core.shape
    q, r, k = qr_colmajor(core.contiguous().view(-1), n * rr, rl)
    return q.view(k, n, rr), r.view(rl, k)  # q^T core, R^T (rl x k)


def _truncated_split_right(core, delta, rmax):
    """Right factor V_r^T and left carry U_r s_r (solver.py:221-236)."""
    rl, n, rr = core.shape
    s, v, k = svd_left_colmajor(core.contiguous().view(-1), n * rr, rl)  # left vectors of M^T
    sh = s.cpu().numpy()
    tail = np.sqrt(np.cumsum(sh[::-1] ** 2))[::-1]
    above = np.nonzero(tail > delta)[0]
    r = int(above[-1] + 1) if above.size else 1
    r = max(1, min(r, rmax))
    vr = v[: (n * rr) * r].view(r, n, rr)  # V[:, :r] column-major == C-order (r, n, rr)
    carry = mm(core.reshape(rl, n * rr), vr.reshape(r, n * rr), tb=True)  # M V_r = U_r s_r
    return vr.contiguous(), carry


def _residual_split_right_structured(core, phi_l, a_p, phi_r, rhs, tol, rmax):
    """_residual_split_right without a dense operator: bisection on r with
    structured local matvecs (the residual of x_r is non-increasing in r up
    to rounding)."""
    rl, n, rr = core.shape
    s, v, k = svd_left_colmajor(core.contiguous().view(-1), n * rr, rl)
    vk = v.view(k, n * rr)
    carry_all = mm(core.reshape(rl, n * rr), vk, tb=True)  # (rl, k) = U S
    bn = float(torch.linalg.vector_norm(rhs))

    def res(r):
        xr = mm(carry_all[:, :r].contiguous(), vk[:r].contiguous()).view(rl, n, rr)
        return float(torch.linalg.vector_norm(_local_matvec(phi_l, a_p, phi_r, xr) - rhs))

    target = max(tol * bn, 2.0 * res(k))
    lo, hi = 1, k  # res(hi) <= target
    while lo < hi:
        mid = (lo + hi) // 2
        if res(mid) <= target:
            hi = mid
        else:
            lo = mid + 1
    r = max(1, min(hi, rmax))
    return vk[:r].contiguous().view(r, n, rr), carry_all[:, :r].contiguous()


def _residual_split_right(core, mcm, rhs, tol, rmax):
    """Local-residual truncation: the smallest r whose truncated core
    x_r = core V_r V_r^T keeps ||M x_r - rhs|| <= max(tol ||rhs||, 2 ||M x - rhs||).
    All candidate residuals come from one GEMM: row i of W is M applied to the
    rank-one increment (core v_i) v_i^T, and x_r's residual is rhs - sum_{i<r} W_i."""
    rl, n, rr = core.shape
    dim = rl * n * rr
    s, v, k = svd_left_colmajor(core.contiguous().view(-1), n * rr, rl)
    vk = v.view(k, n * rr)
    carry_all = mm(core.reshape(rl, n * rr), vk, tb=True)  # (rl, k) = U S
    inc = carry_all.t().unsqueeze(2) * vk.unsqueeze(1)  # (k, rl, n rr)
    w = mm(inc.reshape(k, dim), mcm.view(dim, dim))  # rows: (M inc_i)^T
    resid = rhs.reshape(1, dim) - torch.cumsum(w, dim=0)
    rn = torch.linalg.vector_norm(resid, dim=1).cpu().numpy()
    bn = float(torch.linalg.vector_norm(rhs))
    target = max(tol * bn, 2.0 * rn[-1])
    ok = np.nonzero(rn <= target)[0]
    r = int(ok[0] + 1) if ok.size else k
    r = max(1, min(r, rmax))
    vr = vk[:r].contiguous().view(r, n, rr)
    return vr, carry_all[:, :r].contiguous()


def _safe_core(core, rng):
    if float(torch.linalg.vector_norm(core)) == 0.0:
        return torch.from_numpy(np.asarray(rng.standard_normal(tuple(core.shape))) * 1e-30).to(core.device)
    return core


def _right_orthogonalize_all(cores):
    cores = list(cores)
    for k in range(len(cores) - 1, 0, -1):
        cores[k], carry = _qr_core_right(cores[k])
        cl = cores[k - 1]
        r0, n, r1 = cl.shape
        cores[k - 1] = mm(cl.reshape(r0 * n, r1), carry).view(r0, n, carry.shape[1])
    return cores


def _init_cores(rng, sizes, rank, dev):
    d = len(sizes)
    ranks = [1] + [rank] * (d - 1) + [1]
    host = [rng.standard_normal((ranks[k], sizes[k], ranks[k + 1])) for k in range(d)]
    return _right_orthogonalize_all([torch.from_numpy(c).to(dev) for c in host])


def _operator_views(K: TTMatrix):
    """Per-core permuted copies of the operator cores used by the GEMMs."""
    views = []
    for c in K.device_cores:
        ra, n, m, rb = c.shape
        views.append({
            "ra": ra, "rb": rb, "n": n,
            "a_ijb": c.reshape(ra, n * m * rb),
            "ai_jb": c.reshape(ra * n, m * rb),
            "ib_aj": c.permute(1, 3, 0, 2).reshape(n * rb, ra * m).contiguous(),
            "aj_ib": c.permute(0, 2, 1, 3).reshape(ra * m, n * rb).contiguous(),
        })
    return views


# ------------------------------------------------------------------ solve


def solve(K: TTMatrix, f: TTVector, cfg: SolverConfig, x0: TTVector | None = None) -> SolveOutcome:
    """AMEn-style alternating solve of K u = f (solver.py:239-389).

    ``x0`` (extension, not in the reference API): initial guess replacing the
    seeded rank-2 start; the enrichment cores are still drawn from the seed."""
    if K.col_mode_sizes != f.mode_sizes or K.row_mode_sizes != f.mode_sizes:
        raise ValueError("operator and right-hand side modes do not match")
    t0 = time.perf_counter()
    dev = _lib.device()
    fnorm = tt_norm(f)
    d = f.d
    sizes = f.mode_sizes
    if fnorm == 0.0:
        zero = TTVector([np.zeros((1, n, 1)) for n in sizes])
        return SolveOutcome(zero, 0.0, 0, (1,), (0.0,), time.perf_counter() - t0, True)

    rng = np.random.default_rng(cfg.seed)
    rho = cfg.enrichment_rank
    x = _init_cores(rng, sizes, 2, dev)
    z = _init_cores(rng, sizes, rho, dev)
    if x0 is not None:
        if x0.mode_sizes != sizes:
            raise ValueError("initial guess modes do not match the right-hand side")
        x = _right_orthogonalize_all([c.contiguous().clone() for c in x0.device_cores])
    A = _operator_views(K)
    F = [c.contiguous() for c in f.device_cores]

    one3 = torch.ones((1, 1, 1), dtype=torch.float64, device=dev)
    one2 = torch.ones((1, 1), dtype=torch.float64, device=dev)
    phi_r = [None] * (d + 1)
    psi_r = [None] * (d + 1)
    za_r = [None] * (d + 1)
    zf_r = [None] * (d + 1)
    phi_r[d], psi_r[d], za_r[d], zf_r[d] = one3, one2, one3, one2
    for k in range(d - 1, -1, -1):
        phi_r[k] = _phi_right(phi_r[k + 1], x[k], A[k], x[k])
        psi_r[k] = _psi_right(psi_r[k + 1], x[k], F[k])
        za_r[k] = _phi_right(za_r[k + 1], z[k], A[k], x[k])
        zf_r[k] = _psi_right(zf_r[k + 1], z[k], F[k])
    phi_l = [None] * (d + 1)
    psi_l = [None] * (d + 1)
    za_l = [None] * (d + 1)
    zf_l = [None] * (d + 1)
    phi_l[0], psi_l[0], za_l[0], zf_l[0] = one3, one2, one3, one2

    rank_history, residual_history = [], []
    res, res_prev = np.inf, np.inf
    adapt = 1.0
    residual_rule = cfg.truncation == "residual"
    tol_loc = cfg.trunc_factor * cfg.epsilon / np.sqrt(d)
    sweeps_done = 0
    # With the residual truncation rule nothing in sweep s+1 depends on the
    # residual of sweep s except the decision to stop, so that residual is
    # evaluated on a side stream while sweep s+1 starts; the sweep is
    # abandoned at the next core boundary once the residual shows convergence
    # (the returned u is then the converged iterate of sweep s, exactly as in
    # the sequential order).
    speculate = residual_rule and d <= _DENSE_RESIDUAL_BITS
    pending = None  # (async residual, u, sweep index)
    fd_cache = []
    u_final = None
    best = [np.inf, None, 0, 0]  # best residual, its iterate, its sweep count, sweeps since 2x gain

    def stalled(r, u_it, nsw):
        """Stall rule (cfg.stall_sweeps > 0): True when the residual has not
        halved the best one for stall_sweeps sweeps in a row."""
        if cfg.stall_sweeps <= 0:
            return False
        if r < best[0]:
            gain = r <= 0.5 * best[0]
            best[0], best[1], best[2] = r, u_it, nsw
            if gain:
                best[3] = 0
                return False
        best[3] += 1
        return best[3] >= cfg.stall_sweeps

    def poll(block=False):
        nonlocal pending, res, sweeps_done, u_final
        if pending is None or not (block or pending[0].ready()):
            return False
        ares, pu, ps = pending
        pending = None
        res = ares.value()
        residual_history.append(float(res))
        if _TRACE:
            print(f"[amen] sweep {ps + 1} res {res:.3e} max rank {rank_history[ps]} "
                  f"t {time.perf_counter() - t0:.2f}s", flush=True)
        if res <= cfg.epsilon:
            sweeps_done = ps + 1
            u_final = pu
            return True
        if stalled(res, pu, ps + 1):
            res, u_final, sweeps_done = best[0], best[1], best[2]
            return True
        return False

    for sweep in range(cfg.max_sweeps):
        rtol_local = max(0.02 * cfg.epsilon * adapt, 1e-13)  # solver.py:296
        if residual_rule and cfg.local_rtol_factor > 0.0 and sweep >= 2:
            # residual of sweep s-2: on the speculative path that is the
            # latest one known when sweep s starts (s-1's is still being
            # evaluated), and the sequential path uses the same lag, so both
            # paths follow the same iterates
            rtol_local = max(rtol_local, min(cfg.local_rtol_factor * residual_history[sweep - 2], 1e-4))
        # ---------------- forward: solve + enrich ----------------
        for k in range(d):
            if poll():
                break
            rhs = _local_rhs(psi_l[k], F[k], psi_r[k + 1])
            xk = _solve_local(phi_l[k], A[k], phi_r[k + 1], rhs, x_cur=x[k], cfg=cfg, rtol=rtol_local)
            x[k] = xk
            if k < d - 1:
                zrhs = _local_rhs(zf_l[k], F[k], zf_r[k + 1])
                zloc = zrhs - _proj_a(za_l[k], xk, A[k], za_r[k + 1])
                z[k], _ = _qr_core_left(_safe_core(zloc, rng))
                wrhs = _local_rhs(psi_l[k], F[k], zf_r[k + 1])
                w = wrhs - _proj_a(phi_l[k], xk, A[k], za_r[k + 1])
                xe = torch.cat([x[k], w], dim=2)
                nxt = x[k + 1]
                nxt = torch.cat([nxt, torch.zeros((w.shape[2],) + tuple(nxt.shape[1:]), dtype=torch.float64,
                                                  device=dev)], dim=0)
                with _phase("enrich_qr"):
                    x[k], carry = _qr_core_left(xe)
                r0, n1, r2 = nxt.shape
                x[k + 1] = mm(carry, nxt.reshape(r0, n1 * r2)).view(carry.shape[0], n1, r2)
                with _phase("env"):
                    phi_l[k + 1] = _phi_left(phi_l[k], x[k], A[k], x[k])
                    psi_l[k + 1] = _psi_left(psi_l[k], x[k], F[k])
                    za_l[k + 1] = _phi_left(za_l[k], z[k], A[k], x[k])
                    zf_l[k + 1] = _psi_left(zf_l[k], z[k], F[k])
        if u_final is not None:
            break
        # ---------------- backward: solve + truncate ----------------
        xnorm = float(torch.linalg.vector_norm(x[d - 1]))
        delta = cfg.trunc_factor * cfg.epsilon * adapt * max(xnorm, 1e-300) / np.sqrt(d)
        for k in range(d - 1, -1, -1):
            if poll():
                break
            rhs = _local_rhs(psi_l[k], F[k], psi_r[k + 1])
            xk, mcm = _solve_local(phi_l[k], A[k], phi_r[k + 1], rhs, keep=True, x_cur=x[k], cfg=cfg,
                                   rtol=rtol_local)
            if k > 0:
                with _phase("svd_split"):
                    if residual_rule and mcm is None:
                        x[k], carry = _residual_split_right_structured(xk, phi_l[k], A[k], phi_r[k + 1], rhs,
                                                                      tol_loc, cfg.max_rank)
                    elif residual_rule:
                        x[k], carry = _residual_split_right(xk, mcm, rhs, tol_loc, cfg.max_rank)
                    else:
                        x[k], carry = _truncated_split_right(xk, delta, cfg.max_rank)
                del mcm
                p0, pn, p1 = x[k - 1].shape
                x[k - 1] = mm(x[k - 1].reshape(p0 * pn, p1), carry).view(p0, pn, carry.shape[1])
                with _phase("env"):
                    phi_r[k] = _phi_right(phi_r[k + 1], x[k], A[k], x[k])
                    psi_r[k] = _psi_right(psi_r[k + 1], x[k], F[k])
                    z[k], _ = _qr_core_right(_safe_core(z[k], rng))
                    za_r[k] = _phi_right(za_r[k + 1], z[k], A[k], x[k])
                    zf_r[k] = _psi_right(zf_r[k + 1], z[k], F[k])
            else:
                x[k] = xk
        if u_final is not None or poll(block=True):
            break
        sweeps_done = sweep + 1
        rank_history.append(max(c.shape[0] for c in x[1:]) if d > 1 else 1)
        u = _concat(TTVector, x)
        if speculate and sweep + 1 < cfg.max_sweeps:
            if not fd_cache:
                fd_cache.append(tt_contract_device(f))
            pending = (_AsyncResidual(K, u, fd_cache[0]), u, sweep)
            continue
        with _phase("residual"):
            res = residual(K, u, f)
        residual_history.append(float(res))
        if _TRACE:
            print(f"[amen] sweep {sweep + 1} res {res:.3e} max rank {rank_history[-1]} "
                  f"t {time.perf_counter() - t0:.2f}s", flush=True)
        if res <= cfg.epsilon:
            break
        if stalled(res, u, sweeps_done):
            res, u_final, sweeps_done = best[0], best[1], best[2]
            break
        if not residual_rule and res > 0.7 * res_prev and adapt > 2.0**-44:
            adapt *= 0.25
        res_prev = res

    poll(block=True)
    u = u_final if u_final is not None else _concat(TTVector, x)
    if cfg.stall_sweeps > 0 and best[1] is not None and res > best[0]:
        u, res, sweeps_done = best[1], best[0], best[2]  # best iterate seen
    if cfg.refine_steps > 0 and res > cfg.epsilon and d <= _DENSE_RESIDUAL_BITS:
        u, res = _refine(K, f, u, float(res), cfg, residual_history)
    if res <= cfg.epsilon:
        u, res = _final_compress(K, f, u, res, cfg.epsilon)
    return SolveOutcome(u, float(res), sweeps_done, tuple(rank_history), tuple(residual_history),
                        time.perf_counter() - t0, bool(res <= cfg.epsilon))


def _refine(K, f, u, res, cfg, history):
    """Iterative refinement of a stalled AMEn iterate (SolverConfig.refine_steps)."""
    import dataclasses

    fd = tt_contract_device(f)
    fn = float(torch.linalg.vector_norm(fd))
    for it in range(cfg.refine_steps):
        rd = fd - _apply_tt_to_tt(K, u)
        r_tt = tt_decompose(rd, 0.1 * cfg.refine_tol, mode_sizes=f.mode_sizes)
        del rd
        sub = dataclasses.replace(cfg, epsilon=cfg.refine_tol, refine_steps=0, seed=cfg.seed + 1 + it,
                                  max_sweeps=min(cfg.max_sweeps, 16), stall_sweeps=max(cfg.stall_sweeps, 3))
        corr = solve(K, r_tt, sub)
        # no rounding of u + e: a relative perturbation t of u moves the
        # residual by t ||K|| ||u|| / ||f|| (7e6 t on config 5 at d = 8), so
        # even the _chop floor of tt_round would undo the correction; the
        # sum is only re-rounded if that provably keeps the residual
        cand = tt_add(u, corr.u)
        rc = residual(K, cand, f)
        for fac in (1e-3, 1e-5):
            small = tt_round(cand, fac * cfg.epsilon)
            rs = residual(K, small, f)
            if rs <= 1.1 * rc:
                cand, rc = small, rs
                break
        if _TRACE:
            print(f"[amen] refinement {it + 1}: correction residual {corr.residual:.2e} ({corr.sweeps} sweeps, "
                  f"rhs rank {max(r_tt.ranks)}), residual {res:.3e} -> {rc:.3e}", flush=True)
        if not rc < res:
            break
        gain = res / max(rc, 1e-300)
        u, res = cand, float(rc)
        history.append(res)
        if res <= cfg.epsilon or gain < 4.0:  # converged, or at the FP64 floor of the residual
            break
    return u, res


def _final_compress(K, f, u, res, epsilon):
    """Loosest re-rounding that keeps the residual within epsilon (solver.py:392-409)."""
    if max(epsilon - res, 0.0) <= 0.0:
        return u, res
    # the six candidates are independent: evaluate them concurrently (own
    # stream and host thread each) and keep the first passing one in the
    # reference's order
    def candidate(factor):
        cand = tt_round(u, factor * epsilon)
        return cand, residual(K, cand, f)

    outs = _lib.run_concurrent([(candidate, fac) for fac in (0.5, 0.25, 0.1, 0.03, 0.01, 0.003)])
    for cand, r in outs:
        if r <= epsilon:
            return cand, r
    return u, res
