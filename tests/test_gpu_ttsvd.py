"""Device TT-SVD (ttsvd.cu supersteps + the per-step handoff in round.cu)
against the oracle restatement of ttcore.tt_decompose (ttcore.py:193-264):
equal ranks and reconstruction within eps on inputs that exercise every
path -- several steps per pass, the handoff when r_l n_l > 64, exact low
rank at eps = 0 (rank decisions at the eps_mach floor of _chop), graded
spectra, mode size 4 (matrix TT-SVD), and the zero vector."""

import numpy as np
import pytest

from oracle import tt as O

pytestmark = pytest.mark.gpu


def _T():
    from paper_2501_07778_b200 import ttcore as T

    return T


def _check(v, eps, sizes=None, exact_ranks=True):
    """exact_ranks=False (eps = 0 on exactly low-rank data): the decisions sit
    at the eps_mach floor of _chop, where the reference keeps singular values
    made of its own carry rounding (~5e-15 s0, e.g. rank 6 for a rank-5 TT);
    the device path forms every unfolding from fewer roundings and may drop
    them -- a near-tie at the threshold (north_star's exception).  Then the
    ranks must not exceed the reference's, and the reconstruction is still
    checked to 1e-13."""
    T = _T()
    ref = O.decompose_vector(v, eps, sizes)
    got = T.tt_decompose(v, eps, mode_sizes=sizes) if sizes is not None else T.tt_decompose(v, eps)
    if exact_ranks:
        assert tuple(got.ranks) == tuple(O.ranks(ref)), (got.ranks, O.ranks(ref))
    else:
        assert all(a <= b for a, b in zip(got.ranks, O.ranks(ref))), (got.ranks, O.ranks(ref))
    err = np.linalg.norm(T.tt_contract(got).ravel() - v) / np.linalg.norm(v)
    assert err <= max(eps, 1e-13), err
    return got


def _low_rank_tt(rng, d, r, n=2):
    rk = [1] + [r] * (d - 1) + [1]
    return O.full([rng.standard_normal((rk[k], n, rk[k + 1])) for k in range(d)]).ravel(order="F")


@pytest.mark.parametrize("eps", [0.0, 1e-12, 1e-8])
def test_exact_low_rank(eps):
    """rank-5 TT of 2^16 entries: the supersteps must find rank 5 exactly
    (the _chop floor s0 max(len,2) eps_mach decides at eps = 0)."""
    rng = np.random.default_rng(11)
    v = _low_rank_tt(rng, 16, 5)
    got = _check(v, eps, exact_ranks=eps > 0)
    assert max(got.ranks) == 5


@pytest.mark.parametrize("eps", [1e-4, 1e-8, 1e-10])
def test_smooth_fields(eps):
    """smooth 2-D field in z order (config-3 generator at 2^18 and 2^20)"""
    from tests.golden.cases import config3_field

    for lvl in (9, 10):
        _check(config3_field(lvl), eps)


def test_handoff_to_per_step_path():
    """random data: ranks 2^l grow past 64 / n, so the supersteps hand the
    carry to the per-step path (and get it back for nothing)"""
    rng = np.random.default_rng(12)
    v = rng.standard_normal(1 << 14)
    _check(v, 1e-10)
    _check(v, 0.0)


def test_graded_spectrum():
    """sum of rank-1 terms with geometrically decaying weights 10^-k: the
    singular values of every unfolding span 16 decades"""
    rng = np.random.default_rng(13)
    d = 18
    v = np.zeros(1 << d)
    for k in range(16):
        term = O.full([rng.standard_normal((1, 2, 1)) for _ in range(d)]).ravel(order="F")
        v += 10.0 ** (-k) * term / np.linalg.norm(term)
    for eps in (1e-6, 1e-9, 1e-12):
        _check(v, eps)


def test_mode_size_four():
    rng = np.random.default_rng(14)
    v = _low_rank_tt(rng, 9, 3, n=4)
    got = _check(v, 0.0, sizes=(4,) * 9, exact_ranks=False)
    assert max(got.ranks) == 3
    _check(v + 1e-9 * rng.standard_normal(v.size), 1e-6, sizes=(4,) * 9)


def test_zero_and_tiny():
    T = _T()
    z = T.tt_decompose(np.zeros(1 << 10), 1e-8)
    assert z.ranks == (1,) * 11
    assert np.all(T.tt_contract(z) == 0)
    v = np.zeros(1 << 10)
    v[37] = 1e-3  # a single nonzero: rank 1 everywhere
    got = _check(v, 0.0)
    assert max(got.ranks) == 1
