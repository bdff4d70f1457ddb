"""Canonical and Z-order (Morton) maps: drop-in for ``qttfem.indexing``.

Z = i1 + 2 j1 + 4 i2 + 8 j2 + ... (indexing.py:1-13, 58-64).  The Morton
interleave and the permutations run as device kernels
(``qtt_z_index`` / ``qtt_zorder_permutation`` in libqttb200.so) and are
bit-exact with the reference; results come back as int64 numpy arrays.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

__all__ = [
    "canonical_index",
    "z_index",
    "deinterleave",
    "dof_indices",
    "zorder_permutation",
    "zorder_dof_permutation",
    "permutation_matrix",
]


def _check_range(i, j, d: int) -> None:
    n = 1 << d
    i = np.asarray(i)
    j = np.asarray(j)
    if np.any(i < 0) or np.any(i >= n) or np.any(j < 0) or np.any(j >= n):
        raise ValueError(f"grid index out of range for d={d}: i={i}, j={j}")


def canonical_index(i, j, d: int):
    """Row-major node label L = i + 2^d * j (indexing.py:34-37)."""
    _check_range(i, j, d)
    return i + (1 << d) * j


def z_index(i, j, d: int):
    """Morton label: bit 0 from i, bit 1 from j, ... (indexing.py:58-64)."""
    _check_range(i, j, d)
    ii = np.asarray(i, dtype=np.int64)
    jj = np.asarray(j, dtype=np.int64)
    ii, jj = np.broadcast_arrays(ii, jj)
    dev = _lib.device()
    ti = torch.from_numpy(np.ascontiguousarray(ii).ravel()).to(dev)
    tj = torch.from_numpy(np.ascontiguousarray(jj).ravel()).to(dev)
    out = torch.empty_like(ti)
    _lib.call("qtt_z_index", ctypes.c_int32(d), ctypes.c_int64(ti.numel()), _lib.ptr(ti),
              _lib.ptr(tj), _lib.ptr(out), _lib.stream_handle())
    res = out.cpu().numpy().reshape(ii.shape)
    return res if res.ndim else np.int64(res)


def deinterleave(z, d: int):
    """Recover (i, j) from a Z-order label (indexing.py:67-72)."""
    z = np.asarray(z, dtype=np.int64)
    if np.any(z < 0) or np.any(z >= 1 << (2 * d)):
        raise ValueError(f"z index out of range for d={d}")
    perm = _perm_device(d, False)
    lab = perm[torch.from_numpy(np.ascontiguousarray(z).ravel()).to(perm.device)].cpu().numpy()
    lab = lab.reshape(z.shape)
    mask = (1 << d) - 1
    return lab & mask, lab >> d


def dof_indices(node_index, one_based: bool = False):
    """x/y DOF pair of a node label (indexing.py:75-84)."""
    n = np.asarray(node_index, dtype=np.int64)
    if one_based:
        return 2 * n + 1, 2 * n + 2
    return 2 * n, 2 * n + 1


def _perm_device(d: int, dof: bool) -> torch.Tensor:
    if d < 1:
        raise ValueError("d must be >= 1")
    dev = _lib.device()
    n = (2 if dof else 1) << (2 * d)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    name = "qtt_zorder_dof_permutation" if dof else "qtt_zorder_permutation"
    _lib.call(name, ctypes.c_int32(d), _lib.ptr(out), _lib.stream_handle())
    return out


def zorder_permutation(d: int) -> np.ndarray:
    """``perm[Z_ij] = L_ij`` (indexing.py:87-99), computed on the device."""
    return _perm_device(d, False).cpu().numpy()


def zorder_dof_permutation(d: int) -> np.ndarray:
    """Entry 2Z+c maps to 2L+c (indexing.py:102-112)."""
    return _perm_device(d, True).cpu().numpy()


def permutation_matrix(perm: np.ndarray):
    """Sparse 0/1 matrix P with ``P @ v == v[perm]`` (host helper)."""
    from scipy import sparse

    n = perm.size
    return sparse.csr_matrix((np.ones(n), (np.arange(n), perm)), shape=(n, n))
