"""AMEn-style TT solve on the device: drop-in for ``qttfem.solver``."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .ttcore import TTMatrix, TTVector, tt_contract_device, tt_norm

__all__ = ["SolverConfig", "SolveOutcome", "solve", "residual", "apply_tt_matrix"]

_DENSE_LOCAL_LIMIT = 1200
_DENSE_RESIDUAL_BITS = 22


def apply_tt_matrix(A: TTMatrix, v) -> torch.Tensor:
    """Dense matvec of a TT operator on the device (solver.py:57-73)."""
    dev = _lib.device()
    x = v if isinstance(v, torch.Tensor) else torch.from_numpy(np.asarray(v, dtype=np.float64))
    x = x.to(device=dev, dtype=torch.float64).contiguous()
    out = torch.empty(A.shape[0], dtype=torch.float64, device=dev)
    lay = A._layout()
    _lib.call("qtt_dense_apply", ctypes.byref(lay), _lib.ptr(A.data), _lib.ptr(x), _lib.ptr(out),
              _lib.stream_handle())
    return out
