"""Parity of the device TT algebra (C ABI) against the numpy oracle."""

import numpy as np
import pytest
import torch

from oracle import tt as O

pytestmark = pytest.mark.gpu


def _T():
    from paper_2501_07778_b200 import ttcore as T

    return T


def rand_vec(rng, d, r, n=2):
    rk = [1] + [r] * (d - 1) + [1]
    return [rng.standard_normal((rk[k], n, rk[k + 1])) for k in range(d)]


def rand_mat(rng, d, r, n=2, m=2):
    rk = [1] + [r] * (d - 1) + [1]
    return [rng.standard_normal((rk[k], n, m, rk[k + 1])) for k in range(d)]


def dense_of(t):
    return _T().tt_contract(t)


def _profiled(fn):
    """Run fn with GEMM profiling on; return the dispatch record of its last launch."""
    from paper_2501_07778_b200 import _lib

    _lib.gemm_profile_start()
    try:
        fn()
        torch.cuda.synchronize()
        return _lib.gemm_profile_shapes(1)[0]
    finally:
        _lib.gemm_profile_stop()


def _check_dispatch(rec, path):
    """path: 'tiny' (32x32 tiles), 'tile64' (64x64, no split) or 'split' (64x64, split-K)."""
    if path == "tiny":
        assert rec["bm"] == 32 and rec["splits"] == 1, rec
    elif path == "tile64":
        assert rec["bm"] == 64 and rec["splits"] == 1, rec
    else:
        assert rec["bm"] == 64 and rec["splits"] > 1, rec


@pytest.mark.parametrize("m,n,k,path", [(70, 45, 33, "tiny"), (1000, 700, 96, "tile64"),
                                        (200, 150, 1100, "split")])
def test_gemm_all_transposes(m, n, k, path):
    """All four transpose variants of each kernel configuration (the dispatch
    is asserted from the profiler record, so threshold changes cannot
    silently drop coverage)."""
    T = _T()
    rng = np.random.default_rng(m + n + k)
    for ta in (0, 1):
        for tb in (0, 1):
            a = rng.standard_normal((k, m) if ta else (m, k))
            b = rng.standard_normal((n, k) if tb else (k, n))
            c0 = rng.standard_normal((m, n))
            # column-major buffers: store transposes of C-order arrays
            A = torch.tensor(np.asfortranarray(a).ravel(order="F"), device="cuda")
            B = torch.tensor(np.asfortranarray(b).ravel(order="F"), device="cuda")
            C = torch.tensor(c0.ravel(order="F"), device="cuda")
            rec = _profiled(lambda: T._gemm(ta, tb, m, n, k, 0.5, A, a.shape[0], B, b.shape[0], 2.0, C, m))
            _check_dispatch(rec, path)
            want = 0.5 * (a.T if ta else a) @ (b.T if tb else b) + 2.0 * c0
            got = C.cpu().numpy().reshape((n, m)).T
            assert np.abs(got - want).max() < 1e-12 * np.sqrt(k) * np.abs(want).max()


@pytest.mark.parametrize(
    "m,n,k,ta,flags,path",
    [
        (64, 64, 64, 0, 2 | 4, "tiny"),          # 32x32 tiles, both operands upper triangular
        (512, 512, 512, 0, 4, "tiny"),           # B upper on the 32x32 tiles
        (512, 512, 2048, 0, 4, "split"),         # split-K, B upper (per-chunk K clipping)
        (512, 512, 2048, 0, 2, "split"),         # split-K, A upper
        (512, 512, 2048, 0, 8, "split"),         # split-K, A lower
        (700, 300, 1400, 0, 16, "split"),        # split-K, B lower
        (1024, 1024, 4096, 1, 1, "split"),       # upper-C Gram, split over the computing tiles only
        (2048, 2048, 2048, 0, 2 | 4, "tile64"),  # longest-reduction-first tile order
        (1000, 1000, 1000, 0, 1 | 8 | 4, "split"),  # upper C, A lower, B upper, ragged tiles
        (700, 300, 700, 0, 16, "tiny"),          # B lower triangular
        (1200, 1100, 300, 0, 2 | 16, "tile64"),  # A upper, B lower, 64x64 tiles without split
    ],
)
def test_gemm_structured(m, n, k, ta, flags, path):
    """Structure-flagged DMMA GEMM (upper-C tiles, triangular operand
    clipping, split-K, tile order) against the dense float64 product."""
    rng = np.random.default_rng(m + 7 * n + k + flags)
    a = rng.standard_normal((k, m) if ta else (m, k))
    b = rng.standard_normal((k, n))
    opa = a.T if ta else a
    if flags & 2:
        opa = np.triu(opa)
    if flags & 8:
        opa = np.tril(opa)
    a = opa.T if ta else opa
    if flags & 4:
        b = np.triu(b)
    if flags & 16:
        b = np.tril(b)
    c0 = rng.standard_normal((m, n))
    A = torch.tensor(np.asfortranarray(a).ravel(order="F"), device="cuda")
    B = torch.tensor(np.asfortranarray(b).ravel(order="F"), device="cuda")
    C = torch.tensor(c0.ravel(order="F"), device="cuda")
    from paper_2501_07778_b200 import _lib
    import ctypes

    rec = _profiled(lambda: _lib.call(
        "qtt_gemm_structured", ctypes.c_int32(ta), ctypes.c_int32(0), ctypes.c_int64(m),
        ctypes.c_int64(n), ctypes.c_int64(k), ctypes.c_double(-0.5), _lib.ptr(A),
        ctypes.c_int64(a.shape[0]), _lib.ptr(B), ctypes.c_int64(k), ctypes.c_double(1.5),
        _lib.ptr(C), ctypes.c_int64(m), ctypes.c_int32(flags), _lib.stream_handle()))
    _check_dispatch(rec, path)
    want = -0.5 * opa @ b + 1.5 * c0
    got = C.cpu().numpy().reshape((n, m)).T
    if flags & 1:  # only the upper triangle (incl. diagonal) is specified
        mask = np.triu(np.ones((m, n), dtype=bool))
        got, want = got[mask], want[mask]
    assert np.abs(got - want).max() < 1e-12 * np.sqrt(k) * np.abs(want).max()


@pytest.mark.parametrize("m,n", [(5, 3), (64, 64), (300, 40), (100, 150), (2000, 96), (4100, 70),
                                 (128, 64), (768, 20), (20, 60), (400, 64), (1, 7), (33, 1)])
def test_qr_explicit(m, n):
    from paper_2501_07778_b200 import _lib
    import ctypes

    rng = np.random.default_rng(m + n)
    a = rng.standard_normal((m, n))
    k = min(m, n)
    A = torch.tensor(a.ravel(order="F"), device="cuda")
    Q = torch.zeros(m * k, dtype=torch.float64, device="cuda")
    R = torch.zeros(k * n, dtype=torch.float64, device="cuda")
    _lib.call("qtt_qr", ctypes.c_int64(m), ctypes.c_int64(n), _lib.ptr(A), ctypes.c_int64(m),
              _lib.ptr(Q), ctypes.c_int64(m), _lib.ptr(R), ctypes.c_int64(k), _lib.stream_handle())
    q = Q.cpu().numpy().reshape(k, m).T
    r = R.cpu().numpy().reshape(n, k).T
    assert np.abs(q @ r - a).max() < 1e-12 * np.abs(a).max() * max(m, n) ** 0.5
    assert np.abs(q.T @ q - np.eye(k)).max() < 1e-13 * max(m, n)
    assert np.allclose(np.tril(r, -1), 0.0)


@pytest.mark.parametrize("m,n", [(6, 4), (50, 50), (120, 80), (40, 90), (400, 300)])
def test_svd_values_and_vectors(m, n):
    from paper_2501_07778_b200 import _lib
    import ctypes

    rng = np.random.default_rng(7 * m + n)
    k = min(m, n)
    # graded spectrum down to 1e-14 relative
    u0, _ = np.linalg.qr(rng.standard_normal((m, k)))
    v0, _ = np.linalg.qr(rng.standard_normal((n, k)))
    s0 = np.logspace(0, -14, k)
    a = (u0 * s0) @ v0.T
    A = torch.tensor(a.ravel(order="F"), device="cuda")
    S = torch.zeros(k, dtype=torch.float64, device="cuda")
    U = torch.zeros(m * k, dtype=torch.float64, device="cuda")
    _lib.call("qtt_svd", ctypes.c_int64(m), ctypes.c_int64(n), _lib.ptr(A), ctypes.c_int64(m),
              _lib.ptr(S), _lib.ptr(U), ctypes.c_int64(m), _lib.stream_handle())
    s = S.cpu().numpy()
    s_ref = np.linalg.svd(a, compute_uv=False)
    assert np.abs(s - s_ref).max() <= 1e-14 * s_ref[0] * 10
    u = U.cpu().numpy().reshape(k, m).T
    assert np.abs(u.T @ u - np.eye(k)).max() < 1e-12
    # leading singular subspace matches
    top = 5
    proj = u[:, :top].T @ np.linalg.svd(a)[0][:, :top]
    assert np.allclose(np.abs(np.linalg.svd(proj, compute_uv=False)), 1.0, atol=1e-10)


def test_matvec_matmat_hadamard_add():
    T = _T()
    rng = np.random.default_rng(1)
    A = rand_mat(rng, 6, 3)
    B = rand_mat(rng, 6, 2)
    x = rand_vec(rng, 6, 4)
    y = rand_vec(rng, 6, 2)
    TA, TB, tx, ty = T.TTMatrix(A), T.TTMatrix(B), T.TTVector(x), T.TTVector(y)
    assert np.abs(dense_of(T.tt_matvec(TA, tx)) - O.full(O.matvec(A, x))).max() < 1e-12
    assert np.abs(dense_of(T.tt_matmat(TA, TB)) - O.full(O.matmat(A, B))).max() < 1e-11
    assert np.abs(dense_of(T.tt_hadamard(tx, ty)) - O.full(O.hadamard(x, y))).max() < 1e-12
    assert np.abs(dense_of(T.tt_hadamard(TA, TB)) - O.full(O.hadamard(A, B))).max() < 1e-12
    assert np.abs(dense_of(T.tt_add(tx, ty)) - O.full(O.add(x, y))).max() < 1e-12
    assert np.abs(dense_of(T.tt_add(TA, TB)) - O.full(O.add(A, B))).max() < 1e-12
    assert np.abs(dense_of(T.tt_scale(TA, -2.5)) - O.full(O.scale(A, -2.5))).max() < 1e-12
    assert np.abs(dense_of(T.tt_transpose(TA)) - O.full(A).T).max() < 1e-12
    assert np.abs(dense_of(T.tt_diag(tx)) - np.diag(O.full(x))).max() < 1e-12
    # ranks follow the reference rules
    assert T.tt_matvec(TA, tx).ranks == O.ranks(O.matvec(A, x))
    assert T.tt_add(tx, ty).ranks == O.ranks(O.add(x, y))


def test_zkron_kron_slice():
    T = _T()
    rng = np.random.default_rng(2)
    a, b = rand_vec(rng, 3, 2), rand_vec(rng, 3, 3)
    A, B = rand_mat(rng, 3, 2), rand_mat(rng, 3, 2)
    assert np.abs(dense_of(T.tt_zkron(T.TTVector(a), T.TTVector(b))) - O.full(O.zkron(a, b))).max() < 1e-12
    assert np.abs(dense_of(T.tt_zkron(T.TTMatrix(A), T.TTMatrix(B))) - O.full(O.zkron(A, B))).max() < 1e-12
    assert np.abs(dense_of(T.tt_kron(T.TTMatrix(A), T.TTMatrix(B))) - O.full(O.kron(A, B))).max() < 1e-12
    v = rand_vec(rng, 5, 3)
    for mode in (0, 2, 4):
        got = dense_of(T.tt_slice_mode(T.TTVector(v), mode, 1))
        assert np.abs(got - O.full(O.slice_mode(v, mode, 1))).max() < 1e-12


def test_norm_dot_contract_apply():
    T = _T()
    rng = np.random.default_rng(3)
    x = rand_vec(rng, 8, 5)
    y = rand_vec(rng, 8, 3)
    tx, ty = T.TTVector(x), T.TTVector(y)
    assert abs(T.tt_norm(tx) - np.linalg.norm(O.full(x))) < 1e-12 * np.linalg.norm(O.full(x))
    assert abs(T.tt_dot(tx, ty) - O.full(x) @ O.full(y)) < 1e-11 * np.linalg.norm(O.full(x)) * np.linalg.norm(O.full(y))
    A = rand_mat(rng, 6, 4)
    v = rng.standard_normal(64)
    from paper_2501_07778_b200 import solver

    got = solver.apply_tt_matrix(T.TTMatrix(A), v)
    got = got.cpu().numpy() if hasattr(got, "cpu") else got
    assert np.abs(got - O.full(A) @ v).max() < 1e-11


@pytest.mark.parametrize("eps", [1e-2, 1e-6, 1e-10])
def test_round_ranks_and_error(eps):
    T = _T()
    rng = np.random.default_rng(4)
    for trial in range(6):
        x = rand_vec(rng, 7, 3 + trial % 3)
        z = O.add(O.add(x, O.scale(x, 0.5)), rand_vec(rng, 7, 2))
        ref = O.round_tt(z, eps)
        got = T.tt_round(T.TTVector(z), eps)
        assert got.ranks == O.ranks(ref)
        full = O.full(z)
        err = np.linalg.norm(dense_of(got) - full) / np.linalg.norm(full)
        assert err <= eps * (1 + 1e-8) + 1e-13


@pytest.mark.parametrize("where", ["middle", "late", "none"])
def test_round_speculation_recovers(where):
    """Speculative (sync-free) rounding of a rank-64 TT: full-rank head, then
    an exactly rank-deficient bond in the middle / near the end of the sweep.
    The sticky device flag must send the rounding back to the examined path
    and the result must match the oracle's ranks and values; repeated calls
    give the same bits (the path depends on the input alone)."""
    T = _T()
    d, r = 14, 64
    rng = np.random.default_rng({"middle": 11, "late": 12, "none": 13}[where])
    rk = [1] + [min(r, 2**k, 2 ** (d - k)) for k in range(1, d)] + [1]
    cores = [rng.standard_normal((rk[k], 2, rk[k + 1])) / np.sqrt(rk[k]) for k in range(d)]
    bond = {"middle": 7, "late": 9, "none": None}[where]
    if bond is not None:  # core bond-1 factors through rank 20 (< 64)
        a, n, b = cores[bond - 1].shape
        cores[bond - 1] = (rng.standard_normal((a * n, 20)) @ rng.standard_normal((20, b))).reshape(a, n, b) / 20
    ref = O.round_tt(cores, 1e-10)
    want = O.ranks(ref)
    if bond is not None:
        assert want[bond] == 20
    t = T.TTVector(cores)
    full = O.full(cores)
    first = None
    for rep in range(3):
        got = T.tt_round(t, 1e-10)
        assert got.ranks == want, (rep, got.ranks, want)
        err = np.linalg.norm(dense_of(got) - full) / np.linalg.norm(full)
        assert err <= 1e-10 * (1 + 1e-8) + 1e-13
        if first is None:
            first = got.numpy_cores()
        else:
            assert all(np.array_equal(a, b) for a, b in zip(first, got.numpy_cores()))


@pytest.mark.parametrize("case", ["full", "truncating", "deficient"])
def test_round_streams_cores_to_host(case):
    """tt_round(host=True) (qtt_round_to_host): the cores streamed to pinned
    host memory during the sweep equal the device result bit for bit, for a
    full-rank product, a truncating sum and a rank-deficient input that sends
    the speculative sweep back to the examined path."""
    T = _T()
    rng = np.random.default_rng({"full": 21, "truncating": 22, "deficient": 23}[case])
    if case == "full":
        d, r = 12, 48
        rk = [1] + [min(r, 2**k, 2 ** (d - k)) for k in range(1, d)] + [1]
        cores = [rng.standard_normal((rk[k], 2, rk[k + 1])) for k in range(d)]
    elif case == "truncating":
        x = rand_vec(rng, 9, 5)
        cores = O.add(O.add(x, O.scale(x, 0.25)), rand_vec(rng, 9, 3))
    else:
        d, r = 13, 64
        rk = [1] + [min(r, 2**k, 2 ** (d - k)) for k in range(1, d)] + [1]
        cores = [rng.standard_normal((rk[k], 2, rk[k + 1])) / 8 for k in range(d)]
        a, n, b = cores[6].shape
        cores[6] = (rng.standard_normal((a * n, 9)) @ rng.standard_normal((9, b))).reshape(a, n, b)
    t = T.TTVector(cores)
    full = O.full(cores)
    for rep in range(2):
        dev = T.tt_round(t, 1e-9)
        hst = T.tt_round(t, 1e-9, host=True)
        assert hst.ranks == dev.ranks
        # the streamed host cores are the device cores, bit for bit
        for a, c in zip(hst.cores, hst.numpy_cores()):
            assert isinstance(a, np.ndarray) and not a.flags.writeable
            assert np.array_equal(a, c)
        # and equal to a separate rounding of the same input (the path depends
        # on the input alone)
        for a, b in zip(hst.cores, dev.numpy_cores()):
            assert np.array_equal(a, b)
        got = O.full([np.array(a) for a in hst.cores])
        assert np.linalg.norm(got - full) <= 1e-9 * (1 + 1e-6) * np.linalg.norm(full)


def test_round_matrix():
    T = _T()
    rng = np.random.default_rng(5)
    A = rand_mat(rng, 5, 3)
    z = O.add(A, O.scale(A, 2.0))
    ref = O.round_tt(z, 1e-12)
    got = T.tt_round(T.TTMatrix(z), 1e-12)
    assert got.ranks == O.ranks(ref)
    assert np.abs(dense_of(got) - O.full(z)).max() < 1e-10


@pytest.mark.parametrize("eps", [0.0, 1e-3, 1e-8])
def test_decompose_vector(eps):
    T = _T()
    rng = np.random.default_rng(6)
    xs = np.linspace(0, 1, 1 << 12)
    v = np.sin(3 * xs) * np.exp(-xs) + 0.01 * rng.standard_normal(xs.size) * (eps == 0.0)
    ref = O.decompose_vector(v, eps)
    got = T.tt_decompose(v, eps)
    if eps > 0:
        assert got.ranks == O.ranks(ref)
    err = np.linalg.norm(dense_of(got) - v) / np.linalg.norm(v)
    assert err <= max(eps, 1e-13)


def test_decompose_matrix_and_zero():
    T = _T()
    rng = np.random.default_rng(8)
    m = rng.standard_normal((16, 16))
    got = T.tt_decompose(m, 0.0)
    assert np.abs(dense_of(got) - m).max() < 1e-12
    z = T.tt_decompose(np.zeros(8), 0.0)
    assert z.ranks == (1, 1, 1, 1)


def test_zorder_maps_bit_exact():
    from paper_2501_07778_b200 import indexing

    for d in (1, 3, 6):
        assert np.array_equal(indexing.zorder_permutation(d), O.zorder_permutation(d))
        assert np.array_equal(indexing.zorder_dof_permutation(d), O.zorder_dof_permutation(d))


@pytest.mark.parametrize("m,n", [(150, 150), (300, 277), (277, 400), (420, 420)])
def test_svd_cluster_path(m, n):
    """Mid-size SVDs run the cluster (DSMEM) Jacobi; graded spectra to 1e-13."""
    from paper_2501_07778_b200 import _lib
    import ctypes

    rng = np.random.default_rng(m * 7 + n)
    k = min(m, n)
    u0, _ = np.linalg.qr(rng.standard_normal((m, k)))
    v0, _ = np.linalg.qr(rng.standard_normal((n, k)))
    s0 = np.logspace(0, -13, k)
    a = (u0 * s0) @ v0.T
    A = torch.tensor(a.ravel(order="F"), device="cuda")
    S = torch.zeros(k, dtype=torch.float64, device="cuda")
    U = torch.zeros(m * k, dtype=torch.float64, device="cuda")
    _lib.call("qtt_svd", ctypes.c_int64(m), ctypes.c_int64(n), _lib.ptr(A), ctypes.c_int64(m),
              _lib.ptr(S), _lib.ptr(U), ctypes.c_int64(m), _lib.stream_handle())
    s = S.cpu().numpy()
    assert np.abs(s - np.linalg.svd(a, compute_uv=False)).max() <= 1e-14 * 20
    u = U.cpu().numpy().reshape(k, m).T
    assert np.abs(u.T @ u - np.eye(k)).max() < 1e-12


def test_qr_very_tall_uses_16_wide_panels():
    """m > 16*736 rows switches to 16-column panels (config-5 sized QRs)."""
    from paper_2501_07778_b200 import _lib
    import ctypes

    m, n = 12500, 40
    rng = np.random.default_rng(5)
    a = rng.standard_normal((m, n))
    A = torch.tensor(a.ravel(order="F"), device="cuda")
    Q = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    R = torch.zeros(n * n, dtype=torch.float64, device="cuda")
    _lib.call("qtt_qr", ctypes.c_int64(m), ctypes.c_int64(n), _lib.ptr(A), ctypes.c_int64(m),
              _lib.ptr(Q), ctypes.c_int64(m), _lib.ptr(R), ctypes.c_int64(n), _lib.stream_handle())
    q = Q.cpu().numpy().reshape(n, m).T
    r = R.cpu().numpy().reshape(n, n).T
    assert np.abs(q @ r - a).max() < 1e-11
    assert np.abs(q.T @ q - np.eye(n)).max() < 1e-12


@pytest.mark.parametrize("cond", [1e0, 1e2, 1e3, 1e4, 1e5, 1e6, 1e12])
def test_qr_cholqr_path_and_fallback(cond):
    """n >= 128 tries CholeskyQR2; ill-conditioned inputs fall back to
    Householder.  Both must give an orthonormal Q and A = QR."""
    from paper_2501_07778_b200 import _lib
    import ctypes

    m, n = 1500, 300
    rng = np.random.default_rng(int(np.log10(cond)))
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = (u * np.logspace(0, -np.log10(cond), n)) @ v.T
    A = torch.tensor(a.ravel(order="F"), device="cuda")
    Q = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    R = torch.zeros(n * n, dtype=torch.float64, device="cuda")
    _lib.call("qtt_qr", ctypes.c_int64(m), ctypes.c_int64(n), _lib.ptr(A), ctypes.c_int64(m),
              _lib.ptr(Q), ctypes.c_int64(m), _lib.ptr(R), ctypes.c_int64(n), _lib.stream_handle())
    q = Q.cpu().numpy().reshape(n, m).T
    r = R.cpu().numpy().reshape(n, n).T
    assert np.abs(np.tril(r, -1)).max() == 0.0
    assert np.linalg.norm(q @ r - a) <= 1e-13 * np.linalg.norm(a)
    assert np.abs(q.T @ q - np.eye(n)).max() < 1e-12


@pytest.mark.parametrize("m,n", [(256, 128), (200, 100), (96, 33), (128, 128), (130, 65), (512, 64)])
@pytest.mark.parametrize("cond", [1e0, 1e4, 1e7, 1e13])
def test_qr_small_cholqr_fused(m, n, cond):
    """32 <= n <= 128 runs the sync-free CholeskyQR2 (Gram GEMMs + the fused
    single-CTA factor/inverse kernel, 1 or 2 blocks of 64); ill-conditioned
    inputs raise its status flag and fall back to Householder."""
    from paper_2501_07778_b200 import _lib
    import ctypes

    rng = np.random.default_rng(m + 3 * n + int(np.log10(cond)))
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = (u * np.logspace(0, -np.log10(cond), n)) @ v.T
    A = torch.tensor(a.ravel(order="F"), device="cuda")
    Q = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    R = torch.full((n * n,), 7.0, dtype=torch.float64, device="cuda")
    _lib.call("qtt_qr", ctypes.c_int64(m), ctypes.c_int64(n), _lib.ptr(A), ctypes.c_int64(m),
              _lib.ptr(Q), ctypes.c_int64(m), _lib.ptr(R), ctypes.c_int64(n), _lib.stream_handle())
    q = Q.cpu().numpy().reshape(n, m).T
    r = R.cpu().numpy().reshape(n, n).T
    assert np.abs(np.tril(r, -1)).max() == 0.0
    assert np.linalg.norm(q @ r - a) <= 2e-13 * np.linalg.norm(a)
    assert np.abs(q.T @ q - np.eye(n)).max() < 1e-12


@pytest.mark.parametrize("m,n", [(128, 64), (64, 40), (300, 17)])
def test_qr_small_rank_deficient(m, n):
    """Single-CTA QR with zero / repeated columns (tau = 0 reflectors)."""
    from paper_2501_07778_b200 import _lib
    import ctypes

    rng = np.random.default_rng(m * n)
    a = rng.standard_normal((m, n))
    a[:, 3] = 0.0
    a[:, 5] = a[:, 1]
    a[3:, 7 % n] = 0.0
    k = min(m, n)
    A = torch.tensor(a.ravel(order="F"), device="cuda")
    Q = torch.zeros(m * k, dtype=torch.float64, device="cuda")
    R = torch.zeros(k * n, dtype=torch.float64, device="cuda")
    _lib.call("qtt_qr", ctypes.c_int64(m), ctypes.c_int64(n), _lib.ptr(A), ctypes.c_int64(m),
              _lib.ptr(Q), ctypes.c_int64(m), _lib.ptr(R), ctypes.c_int64(k), _lib.stream_handle())
    q = Q.cpu().numpy().reshape(k, m).T
    r = R.cpu().numpy().reshape(n, k).T
    assert np.abs(q @ r - a).max() < 1e-13 * np.abs(a).max() * m
    assert np.abs(q.T @ q - np.eye(k)).max() < 1e-13 * m
    assert np.allclose(np.tril(r, -1), 0.0)
