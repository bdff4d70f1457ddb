"""Thin wrappers mapping C-order torch matrices onto the column-major C ABI
(DMMA GEMM, Householder QR, Jacobi SVD, dense solve).  Used by the solver's
environment contractions; no arithmetic happens in Python."""

from __future__ import annotations

import ctypes

import torch

from . import _lib


def _S():
    return _lib.stream_handle()


def mm(a: torch.Tensor, b: torch.Tensor, ta: bool = False, tb: bool = False,
       out: torch.Tensor | None = None, alpha: float = 1.0, beta: float = 0.0) -> torch.Tensor:
    """C = alpha op(a) op(b) + beta C for 2-D C-order (contiguous) tensors.

    A C-order (r x c) matrix is the column-major (c x r) matrix in the same
    memory, so C^T = op(b)^T op(a)^T is issued as one column-major GEMM."""
    a = a.contiguous()
    b = b.contiguous()
    m = a.shape[1] if ta else a.shape[0]
    k = a.shape[0] if ta else a.shape[1]
    n = b.shape[0] if tb else b.shape[1]
    kb = b.shape[1] if tb else b.shape[0]
    if k != kb:
        raise ValueError(f"inner dimensions differ: {tuple(a.shape)} {tuple(b.shape)} ta={ta} tb={tb}")
    if out is None:
        out = torch.empty((m, n), dtype=torch.float64, device=a.device)
        beta = 0.0
    _lib.call(
        "qtt_gemm", ctypes.c_int32(1 if tb else 0), ctypes.c_int32(1 if ta else 0), ctypes.c_int64(n),
        ctypes.c_int64(m), ctypes.c_int64(k), ctypes.c_double(alpha), _lib.ptr(b),
        ctypes.c_int64(b.shape[1]), _lib.ptr(a), ctypes.c_int64(a.shape[1]), ctypes.c_double(beta),
        _lib.ptr(out), ctypes.c_int64(n), _S(),
    )
    return out


def qr_colmajor(mat_cm: torch.Tensor, rows: int, cols: int):
    """Householder QR of the column-major (rows x cols) matrix stored in
    ``mat_cm`` (contiguous).  Returns (Q_cm, R_cm) column-major buffers of
    shapes (rows x k) and (k x cols), k = min(rows, cols), as flat tensors."""
    k = min(rows, cols)
    q = torch.empty(rows * k, dtype=torch.float64, device=mat_cm.device)
    r = torch.empty(k * cols, dtype=torch.float64, device=mat_cm.device)
    _lib.call("qtt_qr", ctypes.c_int64(rows), ctypes.c_int64(cols), _lib.ptr(mat_cm),
              ctypes.c_int64(rows), _lib.ptr(q), ctypes.c_int64(rows), _lib.ptr(r), ctypes.c_int64(k), _S())
    return q, r, k


def svd_left_colmajor(mat_cm: torch.Tensor, rows: int, cols: int):
    """Singular values (descending) and left singular vectors (rows x k,
    column-major) of a column-major (rows x cols) matrix."""
    k = min(rows, cols)
    s = torch.empty(k, dtype=torch.float64, device=mat_cm.device)
    u = torch.empty(rows * k, dtype=torch.float64, device=mat_cm.device)
    _lib.call("qtt_svd", ctypes.c_int64(rows), ctypes.c_int64(cols), _lib.ptr(mat_cm),
              ctypes.c_int64(rows), _lib.ptr(s), _lib.ptr(u), ctypes.c_int64(rows), _S())
    return s, u, k


def dense_solve_colmajor(m_cm: torch.Tensor, n: int, b: torch.Tensor) -> tuple:
    """x with M x = b, M column-major (n x n).  Returns (x, used_fallback)."""
    if m_cm.dtype != torch.float64 or b.dtype != torch.float64:
        raise TypeError("dense_solve_colmajor expects float64 tensors")
    x = torch.empty(n, dtype=torch.float64, device=b.device)
    fb = ctypes.c_int32(0)
    b = b.contiguous()
    _lib.call("qtt_dense_solve", ctypes.c_int64(n), _lib.ptr(m_cm.contiguous()), ctypes.c_int64(n),
              _lib.ptr(b), _lib.ptr(x), ctypes.byref(fb), _S())
    return x, bool(fb.value)
