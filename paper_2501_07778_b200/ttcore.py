"""Device tensor trains: drop-in for ``qttfem.ttcore`` (ttcore.py:20-44).

Cores live in ONE packed FP64 CUDA buffer per TT object (core l starts at a
256-byte aligned element offset), in exactly the reference layouts:
vector cores ``(r_{l-1}, n_l, r_l)`` and matrix cores ``(r_{l-1}, n_l, m_l,
r_l)``, flat index LSB-first (ttcore.py:3-10).  Every arithmetic operation
is a call into ``libqttb200.so``; the Python layer validates arguments with
the reference's ValueError/TypeError behaviour, computes output layouts and
owns the buffers.  Objects are immutable; nothing rounds implicitly.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

__all__ = [
    "TTVector",
    "TTMatrix",
    "RankProfile",
    "tt_decompose",
    "tt_contract",
    "tt_round",
    "tt_add",
    "tt_scale",
    "tt_hadamard",
    "tt_matvec",
    "tt_matmat",
    "tt_kron",
    "tt_zkron",
    "tt_transpose",
    "tt_diag",
    "tt_dot",
    "tt_norm",
    "tt_ones",
    "tt_identity",
    "tt_rank1_vector",
    "tt_rank1_matrix",
    "tt_slice_mode",
    "rank_profile",
]

_CONTRACT_GUARD_BITS = 24  # ttcore.py:46


# ------------------------------------------------------------------ layout


def _offsets(shapes) -> tuple:
    off, out = 0, []
    for shp in shapes:
        out.append(off)
        off += _lib.align(int(np.prod(shp)))
    return tuple(out), off


class _TT:
    """Common storage of TTVector / TTMatrix."""

    __slots__ = ("data", "_shapes", "_offs", "_host")
    _order = 3

    def __init__(self, cores):
        arrs = [c for c in cores]
        if not arrs:
            raise ValueError("need at least one core")
        shapes = []
        for c in arrs:
            shp = tuple(int(x) for x in (c.shape if hasattr(c, "shape") else np.shape(c)))
            if len(shp) != self._order:
                kind = "vector" if self._order == 3 else "matrix"
                word = "order-3" if self._order == 3 else "order-4"
                raise ValueError(f"{kind} cores must be {word} arrays")
            shapes.append(shp)
        if shapes[0][0] != 1 or shapes[-1][-1] != 1:
            raise ValueError("boundary ranks must be 1")
        for a, b in zip(shapes[:-1], shapes[1:]):
            if a[-1] != b[0]:
                raise ValueError("adjacent core ranks do not match")
        dev = _lib.device()
        offs, total = _offsets(shapes)
        data = torch.empty(max(total, 1), dtype=torch.float64, device=dev)
        on_host = all(not (isinstance(c, torch.Tensor) and c.is_cuda) for c in arrs)
        if on_host:
            # pack on the host into one pinned staging buffer, one H2D copy
            stage = torch.zeros(max(total, 1), dtype=torch.float64, pin_memory=True)
            sv = stage.numpy()
            for c, shp, o in zip(arrs, shapes, offs):
                a = c.detach().numpy() if isinstance(c, torch.Tensor) else c
                n = int(np.prod(shp))
                sv[o : o + n] = np.asarray(a, dtype=np.float64).reshape(-1)
            data.copy_(stage, non_blocking=True)
        else:
            data.zero_()
            for c, shp, o in zip(arrs, shapes, offs):
                t = c if isinstance(c, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(c, dtype=np.float64))
                n = int(np.prod(shp))
                data[o : o + n].copy_(t.reshape(-1).to(device=dev, dtype=torch.float64), non_blocking=True)
        self.data = data
        self._shapes = tuple(shapes)
        self._offs = offs
        self._host = None

    @classmethod
    def _wrap(cls, data: torch.Tensor, shapes, offs=None):
        obj = cls.__new__(cls)
        obj.data = data
        obj._shapes = tuple(tuple(int(x) for x in s) for s in shapes)
        obj._offs = tuple(offs) if offs is not None else _offsets(obj._shapes)[0]
        obj._host = None
        return obj

    # -------------------------------------------------------------- views
    @property
    def device_cores(self) -> tuple:
        """The cores as CUDA tensor views of the packed buffer (no copy)."""
        return tuple(
            self.data[o : o + int(np.prod(s))].view(s) for o, s in zip(self._offs, self._shapes)
        )

    @property
    def cores(self) -> tuple:
        """The cores as read-only host numpy arrays, like the reference's
        frozen cores (ttcore.py:49-52,61,71): one D2H copy on first access,
        cached (the object is immutable).  Device code uses device_cores."""
        host = getattr(self, "_host", None)
        if host is None:
            host = tuple(self.numpy_cores())
            for a in host:
                a.flags.writeable = False
            self._host = host
        return host

    def numpy_cores(self) -> list:
        """Host copies of the cores: one D2H copy of the packed buffer into
        pinned memory, returned as numpy views of it."""
        # only the used extent: results of tt_round / tt_decompose live in
        # input-sized buffers that can be much larger than the rounded cores
        end = max((o + int(np.prod(s)) for o, s in zip(self._offs, self._shapes)), default=0)
        host = torch.empty(max(end, 1), dtype=torch.float64, pin_memory=True)
        host[:end].copy_(self.data[:end])
        hv = host.numpy()
        return [hv[o : o + int(np.prod(s))].reshape(s) for o, s in zip(self._offs, self._shapes)]

    @property
    def d(self) -> int:
        return len(self._shapes)

    @property
    def ranks(self) -> tuple:
        return (1,) + tuple(s[-1] for s in self._shapes)

    def _layout(self) -> _lib.Layout:
        lay = _lib.Layout()
        lay.d = self.d
        lay.is_matrix = 1 if self._order == 4 else 0
        lay.ranks[0] = 1
        for l, s in enumerate(self._shapes):
            lay.ranks[l + 1] = s[-1]
            lay.rows[l] = s[1]
            lay.cols[l] = s[2] if self._order == 4 else 1
            lay.offsets[l] = self._offs[l]
        return lay


class TTVector(_TT):
    """Tensor train with order-3 cores of shape (r_{l-1}, n_l, r_l)."""

    __slots__ = ()
    _order = 3

    @property
    def mode_sizes(self) -> tuple:
        return tuple(s[1] for s in self._shapes)

    @property
    def size(self) -> int:
        return int(np.prod(self.mode_sizes, dtype=np.int64))

    def __repr__(self):
        return f"TTVector(modes={self.mode_sizes}, ranks={self.ranks})"


class TTMatrix(_TT):
    """Tensor train operator with order-4 cores (r_{l-1}, n_l, m_l, r_l)."""

    __slots__ = ()
    _order = 4

    @property
    def row_mode_sizes(self) -> tuple:
        return tuple(s[1] for s in self._shapes)

    @property
    def col_mode_sizes(self) -> tuple:
        return tuple(s[2] for s in self._shapes)

    @property
    def shape(self) -> tuple:
        return (
            int(np.prod(self.row_mode_sizes, dtype=np.int64)),
            int(np.prod(self.col_mode_sizes, dtype=np.int64)),
        )

    def __repr__(self):
        return f"TTMatrix(rows={self.row_mode_sizes}, cols={self.col_mode_sizes}, ranks={self.ranks})"


class RankProfile:
    """Rank and storage statistics of one TT object (ttcore.py:141-156)."""

    __slots__ = ("max_rank", "param_count", "storage_count", "effective_rank")

    def __init__(self, max_rank, param_count, storage_count, effective_rank):
        self.max_rank = int(max_rank)
        self.param_count = int(param_count)
        self.storage_count = int(storage_count)
        self.effective_rank = float(effective_rank)

    def __repr__(self):
        return (
            f"RankProfile(R={self.max_rank}, N={self.param_count}, "
            f"storage={self.storage_count}, erank={self.effective_rank:.3f})"
        )


# ----------------------------------------------------------------- helpers


def _is_tt(t) -> bool:
    return isinstance(t, (TTVector, TTMatrix))


def _new_like(kind, shapes):
    offs, total = _offsets(shapes)
    data = torch.empty(max(total, 1), dtype=torch.float64, device=_lib.device())
    return kind._wrap(data, shapes, offs)


def _from_layout(kind, lay: _lib.Layout, data: torch.Tensor):
    shapes = []
    for l in range(lay.d):
        r0, r1 = lay.ranks[l], lay.ranks[l + 1]
        if kind is TTMatrix:
            shapes.append((r0, lay.rows[l], lay.cols[l], r1))
        else:
            shapes.append((r0, lay.rows[l], r1))
    return kind._wrap(data, shapes, [lay.offsets[l] for l in range(lay.d)])


def _check_same_modes(a, b):
    if isinstance(a, TTVector) != isinstance(b, TTVector):
        raise ValueError("cannot mix vectors and matrices")
    if isinstance(a, TTVector):
        if a.mode_sizes != b.mode_sizes:
            raise ValueError("mode-size mismatch")
    elif a.row_mode_sizes != b.row_mode_sizes or a.col_mode_sizes != b.col_mode_sizes:
        raise ValueError("mode-size mismatch")


def _S():
    return _lib.stream_handle()


# ------------------------------------------------------------------ TT-SVD


def tt_decompose(dense, epsilon: float, mode_sizes=None):
    """TT-SVD of a dense vector (1-D) or square matrix (2-D) on the device
    (ttcore.py:211-264).  ``dense`` may be a numpy array or a torch tensor
    (host or device)."""
    if epsilon < 0:
        raise ValueError("epsilon must be >= 0")
    dev = _lib.device()
    x = dense if isinstance(dense, torch.Tensor) else torch.from_numpy(np.asarray(dense, dtype=np.float64))
    x = x.to(device=dev, dtype=torch.float64)
    if x.dim() == 1:
        n = x.numel()
        if mode_sizes is None:
            d = int(n).bit_length() - 1
            if n != (1 << d) or n < 2:
                raise ValueError(f"vector length {n} is not a power of two")
            mode_sizes = (2,) * d
        mode_sizes = tuple(int(m) for m in mode_sizes)
        if int(np.prod(mode_sizes)) != n:
            raise ValueError("mode sizes do not match vector length")
        return _decompose_vec(x.contiguous(), mode_sizes, epsilon)
    if x.dim() == 2:
        nr, nc = x.shape
        if mode_sizes is None:
            d = int(nr).bit_length() - 1
            if nr != (1 << d) or nc != nr or nr < 2:
                raise ValueError(f"matrix shape {tuple(x.shape)} is not square power-of-two")
            rows = cols = (2,) * d
        else:
            rows, cols = mode_sizes
        rows, cols = tuple(int(v) for v in rows), tuple(int(v) for v in cols)
        if int(np.prod(rows)) != nr or int(np.prod(cols)) != nc:
            raise ValueError("mode sizes do not match matrix shape")
        d = len(rows)
        flat = _matrix_to_merged(x.contiguous(), rows, cols)
        vec = _decompose_vec(flat, tuple(rows[l] * cols[l] for l in range(d)), epsilon)
        shapes = [(sh[0], rows[l], cols[l], sh[2]) for l, sh in enumerate(vec._shapes)]
        return TTMatrix._wrap(vec.data, shapes, vec._offs)
    raise ValueError("dense input must be 1D or 2D")


def _matrix_to_merged(x: torch.Tensor, rows, cols) -> torch.Tensor:
    """Dense (R x C) matrix -> merged vector v[K], K = sum_l (i_l m_l + j_l) prod_{t<l} n_t m_t."""
    d = len(rows)
    # x[I, J] with I = sum i_l prod n, J = sum j_l prod m (LSB first).  As a
    # C-order tensor: x.reshape(rows reversed + cols reversed)
    t = x.reshape(tuple(reversed(rows)) + tuple(reversed(cols)))
    # axis of i_l is d-1-l, axis of j_l is 2d-1-l; target C-order axes from
    # slowest merged mode to fastest: (i_{d-1}, j_{d-1}, ..., i_0, j_0)
    order = []
    for l in reversed(range(d)):
        order += [d - 1 - l, 2 * d - 1 - l]
    return t.permute(*order).contiguous().reshape(-1)


def _decompose_vec(x: torch.Tensor, sizes, epsilon) -> TTVector:
    d = len(sizes)
    cap = 3 * x.numel() + 64 * d + 64
    out = torch.empty(cap, dtype=torch.float64, device=x.device)
    lay = _lib.Layout()
    arr = (ctypes.c_int64 * d)(*sizes)
    _lib.call("qtt_decompose", _lib.ptr(x), ctypes.c_int32(d), arr, ctypes.c_double(epsilon),
              ctypes.byref(lay), _lib.ptr(out), ctypes.c_int64(cap), _S())
    return _from_layout(TTVector, lay, out)


# ----------------------------------------------------------------- dense


def tt_contract_device(t) -> torch.Tensor:
    """Dense realisation on the device (ttcore.py:267-293)."""
    if isinstance(t, TTVector):
        bits = sum(int(n).bit_length() - 1 if n > 1 else 1 for n in t.mode_sizes)
        if t.d > _CONTRACT_GUARD_BITS or bits > _CONTRACT_GUARD_BITS:
            raise ValueError(f"refusing to materialize vector with d={t.d}")
        out = torch.empty(t.size, dtype=torch.float64, device=t.data.device)
        lay = t._layout()
        _lib.call("qtt_contract", ctypes.byref(lay), _lib.ptr(t.data), _lib.ptr(out), _S())
        return out
    if isinstance(t, TTMatrix):
        if t.d > _CONTRACT_GUARD_BITS // 2:
            raise ValueError(f"refusing to materialize matrix with d={t.d}")
        nr, nc = t.shape
        out = torch.empty(nr * nc, dtype=torch.float64, device=t.data.device)
        lay = t._layout()
        _lib.call("qtt_contract", ctypes.byref(lay), _lib.ptr(t.data), _lib.ptr(out), _S())
        # kernel writes column-major (I fastest): return a (nr, nc) view
        return out.view(nc, nr).t()
    raise TypeError(f"not a TT object: {type(t)}")


def tt_contract(t) -> np.ndarray:
    """Dense realisation as a host numpy array (reference return type)."""
    return tt_contract_device(t).cpu().numpy()


# ------------------------------------------------------------- rounding


def tt_round(t, epsilon: float, host: bool = False):
    """Compress at relative tolerance epsilon; ranks never increase
    (ttcore.py:322-338).

    ``host=True`` (extension): the cores are also streamed to pinned host
    memory while the sweep runs (``qtt_round_to_host``), so ``.cores`` of the
    result -- host arrays, as the reference returns them -- costs no separate
    device-to-host pass."""
    if epsilon < 0:
        raise ValueError("epsilon must be >= 0")
    if not _is_tt(t):
        raise TypeError(f"not a TT object: {type(t)}")
    lay = t._layout()
    out_lay = _lib.Layout()
    out = torch.empty_like(t.data)
    if not host:
        _lib.call("qtt_round", ctypes.byref(lay), _lib.ptr(t.data), ctypes.c_double(epsilon),
                  ctypes.byref(out_lay), _lib.ptr(out), _S())
        return _from_layout(type(t), out_lay, out)
    # ranks never exceed the structural bounds: a tight capacity for the pinned buffer
    ranks = list(t.ranks)
    sizes = [int(np.prod(s[1:-1])) for s in t._shapes]
    left = right = 1
    for k in range(1, len(ranks) - 1):
        left *= sizes[k - 1]
        ranks[k] = min(ranks[k], left)
    for k in range(len(ranks) - 2, 0, -1):
        right *= sizes[k]
        ranks[k] = min(ranks[k], right)
    cap = sum(_lib.align(ranks[k] * sizes[k] * ranks[k + 1]) for k in range(len(sizes)))
    hbuf = torch.empty(max(cap, 1), dtype=torch.float64, pin_memory=True)
    _lib.call("qtt_round_to_host", ctypes.byref(lay), _lib.ptr(t.data), ctypes.c_double(epsilon),
              ctypes.byref(out_lay), _lib.ptr(out), ctypes.c_void_p(hbuf.data_ptr()), _S())
    res = _from_layout(type(t), out_lay, out)
    hv = hbuf.numpy()
    cores = tuple(hv[o : o + int(np.prod(s))].reshape(s) for o, s in zip(res._offs, res._shapes))
    for a in cores:
        a.flags.writeable = False
    res._host = cores
    return res


def tt_norm(t) -> float:
    """Frobenius/Euclidean norm (after right-to-left orthogonalisation)."""
    if not _is_tt(t):
        raise TypeError(f"not a TT object: {type(t)}")
    res = ctypes.c_double(0.0)
    lay = t._layout()
    _lib.call("qtt_norm", ctypes.byref(lay), _lib.ptr(t.data), ctypes.byref(res), _S())
    return float(res.value)


def tt_dot(a: TTVector, b: TTVector) -> float:
    """Inner product <a, b> (ttcore.py:355-363)."""
    if a.mode_sizes != b.mode_sizes:
        raise ValueError("mode-size mismatch in dot product")
    res = ctypes.c_double(0.0)
    la, lb = a._layout(), b._layout()
    _lib.call("qtt_dot", ctypes.byref(la), _lib.ptr(a.data), ctypes.byref(lb), _lib.ptr(b.data),
              ctypes.byref(res), _S())
    return float(res.value)


# --------------------------------------------------------- structural ops


def tt_add(a, b):
    """Elementwise sum; ranks add (ttcore.py:380-411)."""
    _check_same_modes(a, b)
    return _add_scaled(a, b, 1.0)


def _add_scaled(a, b, beta: float):
    d = a.d
    shapes = []
    for k, (sa, sb) in enumerate(zip(a._shapes, b._shapes)):
        r0 = 1 if k == 0 else sa[0] + sb[0]
        r1 = 1 if k == d - 1 else sa[-1] + sb[-1]
        shapes.append((r0,) + sa[1:-1] + (r1,))
    out = _new_like(type(a), shapes)
    la, lb, lc = a._layout(), b._layout(), out._layout()
    _lib.call("qtt_add", ctypes.byref(la), _lib.ptr(a.data), ctypes.byref(lb), _lib.ptr(b.data),
              ctypes.c_double(beta), ctypes.byref(lc), _lib.ptr(out.data), _S())
    return out


def tt_sub(a, b):
    """a - b in one launch (rank concatenation with the second block negated)."""
    _check_same_modes(a, b)
    return _add_scaled(a, b, -1.0)


def tt_scale(a, s: float):
    """Scalar multiple: core 0 scaled (ttcore.py:414-418)."""
    if not _is_tt(a):
        raise TypeError(f"not a TT object: {type(a)}")
    out = type(a)._wrap(torch.empty_like(a.data), a._shapes, a._offs)
    lay = a._layout()
    _lib.call("qtt_scale", ctypes.byref(lay), _lib.ptr(a.data), ctypes.c_double(float(s)),
              _lib.ptr(out.data), _S())
    return out


def tt_hadamard(a, b):
    """Elementwise product; ranks multiply (ttcore.py:421-440)."""
    _check_same_modes(a, b)
    shapes = [
        (sa[0] * sb[0],) + sa[1:-1] + (sa[-1] * sb[-1],) for sa, sb in zip(a._shapes, b._shapes)
    ]
    out = _new_like(type(a), shapes)
    la, lb, lc = a._layout(), b._layout(), out._layout()
    _lib.call("qtt_hadamard", ctypes.byref(la), _lib.ptr(a.data), ctypes.byref(lb),
              _lib.ptr(b.data), ctypes.byref(lc), _lib.ptr(out.data), _S())
    return out


def tt_matvec(A: TTMatrix, x: TTVector) -> TTVector:
    """Exact product A @ x, all cores in one launch (ttcore.py:443-455)."""
    if A.col_mode_sizes != x.mode_sizes:
        raise ValueError("mode-size mismatch in matvec")
    shapes = [(sa[0] * sx[0], sa[1], sa[3] * sx[2]) for sa, sx in zip(A._shapes, x._shapes)]
    out = _new_like(TTVector, shapes)
    la, lx, ly = A._layout(), x._layout(), out._layout()
    _lib.call("qtt_matvec", ctypes.byref(la), _lib.ptr(A.data), ctypes.byref(lx),
              _lib.ptr(x.data), ctypes.byref(ly), _lib.ptr(out.data), _S())
    return out


def tt_matmat(A: TTMatrix, B: TTMatrix) -> TTMatrix:
    """Exact product A @ B (ttcore.py:458-470)."""
    if A.col_mode_sizes != B.row_mode_sizes:
        raise ValueError("mode-size mismatch in matmat")
    shapes = [
        (sa[0] * sb[0], sa[1], sb[2], sa[3] * sb[3]) for sa, sb in zip(A._shapes, B._shapes)
    ]
    out = _new_like(TTMatrix, shapes)
    la, lb, lc = A._layout(), B._layout(), out._layout()
    _lib.call("qtt_matmat", ctypes.byref(la), _lib.ptr(A.data), ctypes.byref(lb),
              _lib.ptr(B.data), ctypes.byref(lc), _lib.ptr(out.data), _S())
    return out


def tt_transpose(A: TTMatrix) -> TTMatrix:
    shapes = [(s[0], s[2], s[1], s[3]) for s in A._shapes]
    out = _new_like(TTMatrix, shapes)
    la, lt = A._layout(), out._layout()
    _lib.call("qtt_transpose", ctypes.byref(la), _lib.ptr(A.data), ctypes.byref(lt),
              _lib.ptr(out.data), _S())
    return out


def tt_diag(v: TTVector) -> TTMatrix:
    """Diagonal operator with the entries of v (ttcore.py:478-486)."""
    shapes = [(s[0], s[1], s[1], s[2]) for s in v._shapes]
    out = _new_like(TTMatrix, shapes)
    lv, ld = v._layout(), out._layout()
    _lib.call("qtt_diag", ctypes.byref(lv), _lib.ptr(v.data), ctypes.byref(ld),
              _lib.ptr(out.data), _S())
    return out


def tt_kron(A, B):
    """Kronecker product, B's cores first (ttcore.py:489-498)."""
    if isinstance(A, TTVector) != isinstance(B, TTVector):
        raise ValueError("cannot mix vectors and matrices")
    return _concat(type(A), list(B.device_cores) + list(A.device_cores))


def _concat(kind, cores):
    shapes = [tuple(c.shape) for c in cores]
    out = _new_like(kind, shapes)
    for c, o, s in zip(cores, out._offs, shapes):
        n = int(np.prod(s))
        out.data[o : o + n].copy_(c.reshape(-1))
    return out


def tt_zkron(A, B):
    """Bit-interleaved Kronecker product (ttcore.py:501-539)."""
    if isinstance(A, TTVector) != isinstance(B, TTVector):
        raise ValueError("cannot mix vectors and matrices")
    if A.d != B.d:
        raise ValueError("z-kron factors must have matching depth")
    shapes = []
    for sa, sb in zip(A._shapes, B._shapes):
        ra0, ra1, rb0, rb1 = sa[0], sa[-1], sb[0], sb[-1]
        shapes.append((rb0 * ra0,) + sb[1:-1] + (rb1 * ra0,))
        shapes.append((rb1 * ra0,) + sa[1:-1] + (rb1 * ra1,))
    out = _new_like(type(A), shapes)
    la, lb, lc = A._layout(), B._layout(), out._layout()
    _lib.call("qtt_zkron", ctypes.byref(la), _lib.ptr(A.data), ctypes.byref(lb),
              _lib.ptr(B.data), ctypes.byref(lc), _lib.ptr(out.data), _S())
    return out


# --------------------------------------------------------- constructors


def tt_ones(mode_sizes) -> TTVector:
    return TTVector([np.ones((1, n, 1)) for n in mode_sizes])


def tt_identity(mode_sizes) -> TTMatrix:
    return TTMatrix([np.eye(n).reshape(1, n, n, 1) for n in mode_sizes])


def tt_rank1_vector(factors) -> TTVector:
    """Rank-1 TT from per-mode 1-D factors (first varies fastest)."""
    return TTVector([np.asarray(f, float).reshape(1, -1, 1) for f in factors])


def tt_rank1_matrix(factors) -> TTMatrix:
    out = []
    for f in factors:
        f = np.asarray(f, float)
        out.append(f.reshape(1, f.shape[0], f.shape[1], 1))
    return TTMatrix(out)


def tt_slice_mode(t, mode: int, index: int):
    """Fix one mode and absorb it into a neighbour (ttcore.py:566-586)."""
    if isinstance(t, TTMatrix):
        raise TypeError("mode slicing is defined for vectors")
    if not isinstance(t, TTVector):
        raise TypeError(f"not a TT object: {type(t)}")
    if not 0 <= mode < t.d:
        raise ValueError("mode out of range")
    if t.d == 1:
        raise ValueError("cannot slice away the only mode")
    cores = list(t.device_cores)
    sl = cores[mode][:, index, :].contiguous()  # (r0, r1)
    del cores[mode]
    if mode == 0:
        nb = cores[0]
        r0, n, r2 = nb.shape
        newc = torch.empty((sl.shape[0], n, r2), dtype=torch.float64, device=nb.device)
        # new (1 x n r2) row-major = sl (1 x r0) @ nb (r0 x n r2); column-major:
        # new^T (n r2 x 1) = nb^T (n r2 x r0) @ sl^T (r0 x 1)
        _gemm(0, 0, n * r2, sl.shape[0], r0, 1.0, nb, n * r2, sl, r0, 0.0, newc, n * r2)
        cores[0] = newc
    else:
        pc = cores[mode - 1]
        r0, n, r1 = pc.shape
        r2 = sl.shape[1]
        newc = torch.empty((r0, n, r2), dtype=torch.float64, device=pc.device)
        # new (r0 n x r2) row-major = pc (r0 n x r1) @ sl (r1 x r2); column-major:
        # new^T (r2 x r0 n) = sl^T (r2 x r1) @ pc^T (r1 x r0 n)
        _gemm(0, 0, r2, r0 * n, r1, 1.0, sl, r2, pc, r1, 0.0, newc, r2)
        cores[mode - 1] = newc
    return _concat(TTVector, cores)


def _gemm(ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc):
    """Column-major C = alpha op(A) op(B) + beta C through qtt_gemm."""
    _lib.call("qtt_gemm", ctypes.c_int32(ta), ctypes.c_int32(tb), ctypes.c_int64(m),
              ctypes.c_int64(n), ctypes.c_int64(k), ctypes.c_double(alpha), _lib.ptr(a),
              ctypes.c_int64(lda), _lib.ptr(b), ctypes.c_int64(ldb), ctypes.c_double(beta),
              _lib.ptr(c), ctypes.c_int64(ldc), _S())


# ------------------------------------------------------------- profiling


def _erank(mode_sizes, storage: int) -> float:
    d = len(mode_sizes)
    if d == 1:
        return storage / mode_sizes[0]
    a = float(sum(mode_sizes[1:-1]))
    b = float(mode_sizes[0] + mode_sizes[-1])
    if a == 0.0:
        return storage / b
    return (-b + np.sqrt(b * b + 4.0 * a * storage)) / (2.0 * a)


def rank_profile(t) -> RankProfile:
    """Max rank, stored-scalar count and effective rank (ttcore.py:589-613)."""
    sizes = [int(np.prod(s[1:-1])) for s in t._shapes]
    storage = sum(int(np.prod(s)) for s in t._shapes)
    ranks = [s[-1] for s in t._shapes[:-1]]
    return RankProfile(max(ranks) if ranks else 1, storage, storage, _erank(sizes, storage))
