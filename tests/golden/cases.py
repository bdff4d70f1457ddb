"""Seeded inputs shared by the golden generator and the tests."""

from __future__ import annotations

import numpy as np

UNIT = [[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]]
TRAPEZOID = [[0.0, 0.0], [1.1, 0.0], [1.3, 1.2], [0.0, 0.9]]


def _vec(rng, d, r, n=2):
    rk = [1] + [r] * (d - 1) + [1]
    return [rng.standard_normal((rk[k], n, rk[k + 1])) for k in range(d)]


def _mat(rng, d, r):
    rk = [1] + [r] * (d - 1) + [1]
    return [rng.standard_normal((rk[k], 2, 2, rk[k + 1])) for k in range(d)]


def tt_cases():
    out = {}
    for seed, (d, ra, rb, rx, ry) in enumerate([(4, 2, 3, 3, 2), (6, 3, 2, 4, 5), (8, 2, 2, 3, 3)]):
        rng = np.random.default_rng(100 + seed)
        out[f"c{seed}"] = (_mat(rng, d, ra), _vec(rng, d, rx), _mat(rng, d, rb), _vec(rng, d, ry))
    return out


def config2_small(rA, rx, d):
    """Config-2 generator at a reduced depth."""
    rng_a = np.random.default_rng(1000 + rA)
    ra = [1] + [rA] * (d - 1) + [1]
    A = [rng_a.standard_normal((ra[k], 2, 2, ra[k + 1])) / np.sqrt(rA) for k in range(d)]
    rng_x = np.random.default_rng(2000 + rx)
    rc = [1] + [rx] * (d - 1) + [1]
    x = [rng_x.standard_normal((rc[k], 2, rc[k + 1])) / np.sqrt(rx) for k in range(d)]
    return A, x


def config3_round(d=12, terms=16, r=2):
    """Config-3 rounding generator (16 random rank-r terms) at reduced size."""
    rng = np.random.default_rng(3000)
    acc = None
    for _ in range(terms):
        rk = [1] + [r] * (d - 1) + [1]
        t = [rng.standard_normal((rk[k], 2, rk[k + 1])) / np.sqrt(r) for k in range(d)]
        if acc is None:
            acc = t
        else:
            new = []
            for k, (a, b) in enumerate(zip(acc, t)):
                r0 = 1 if k == 0 else a.shape[0] + b.shape[0]
                r1 = 1 if k == d - 1 else a.shape[2] + b.shape[2]
                c = np.zeros((r0, 2, r1))
                o0 = 0 if k == 0 else a.shape[0]
                o1 = 0 if k == d - 1 else a.shape[2]
                c[: a.shape[0], :, : a.shape[2]] = a
                c[o0 : o0 + b.shape[0], :, o1 : o1 + b.shape[2]] += b
                new.append(c)
            acc = new
    return acc


def config3_field(bits=5):
    """g(x,y) = sin(3x) exp(-y) + 0.1 cos(7xy) on a 2^bits grid, Z-ordered."""
    n = 1 << bits
    xs = np.arange(n) / (n - 1)
    X, Y = np.meshgrid(xs, xs, indexing="ij")
    g = np.sin(3 * X) * np.exp(-Y) + 0.1 * np.cos(7 * X * Y)
    t = g.reshape((2,) * (2 * bits), order="F")
    t = t.transpose([ax for k in range(bits) for ax in (k, bits + k)])
    return t.ravel(order="F")


def round_cases():
    out = {}
    rng = np.random.default_rng(5)
    x = _vec(rng, 7, 3)
    y = _vec(rng, 7, 2)
    from oracle import tt as O  # pure numpy helpers to build inputs

    out["sum_1e-6"] = (O.add(O.add(x, O.scale(x, 0.5)), y), 1e-6)
    out["sum_1e-12"] = (O.add(O.add(x, O.scale(x, 0.5)), y), 1e-12)
    A, xx = config2_small(4, 4, 10)
    out["c2_d10"] = (O.matvec(A, xx), 1e-10)
    out["c3_d12_1e-6"] = (config3_round(), 1e-6)
    out["c3_d12_1e-10"] = (config3_round(), 1e-10)
    M = _mat(rng, 5, 3)
    out["mat"] = (O.add(M, O.scale(M, 2.0)), 1e-12)
    return out


def decompose_cases():
    rng = np.random.default_rng(6)
    xs = np.linspace(0, 1, 1 << 12)
    return {
        "smooth_1e-8": (np.sin(3 * xs) * np.exp(-xs), 1e-8),
        "noise_0": (rng.standard_normal(256), 0.0),
        "field5_1e-8": (config3_field(5), 1e-8),
        "field6_1e-6": (config3_field(6), 1e-6),
    }


def apply_case():
    rng = np.random.default_rng(9)
    return _mat(rng, 6, 3)


def element_cases():
    return {
        "trap2": {"corners": TRAPEZOID, "d": 2, "material": (1.0, 0.3, "plane-stress")},
        "unit3": {"corners": UNIT, "d": 3, "material": (2.0, 0.25, "plane-strain")},
    }


def assembly_cases():
    return {
        "unit2": {"corners": UNIT, "d": 2, "material": (64.0, 0.0, "plane-stress"), "ordering": "zorder",
                  "eps": 1e-12, "body": (0.0, 0.0)},
        "unit3b": {"corners": UNIT, "d": 3, "material": (1.0, 0.3, "plane-stress"), "ordering": "zorder",
                   "eps": 1e-8, "body": (0.0, -1.0)},
        "trap3": {"corners": TRAPEZOID, "d": 3, "material": (1.0, 0.3, "plane-strain"), "ordering": "zorder",
                  "eps": 1e-10, "body": (0.5, -1.0)},
        "trap2c": {"corners": TRAPEZOID, "d": 2, "material": (1.0, 0.3, "plane-stress"), "ordering": "canonical",
                   "eps": 1e-12, "body": (0.0, -1.0)},
    }


def shift_cases():
    return {"d3o0": (3, 0), "d3o1": (3, 1), "d1o1": (1, 1), "d4o1": (4, 1)}


def coupling_cases():
    shifted = lambda dx, dy: [[x + dx, y + dy] for x, y in UNIT]  # noqa: E731
    return {
        "single3": {
            "meshes": [{"corners": UNIT, "d": 3, "tags": {"left": "clamped"}, "tractions": {"right": (1.0, 0.0)}}],
            "material": (1.0, 0.3, "plane-stress"), "eps": 1e-8, "body": (0.0, 0.0), "solve": 1e-8,
        },
        "lshape2": {
            "meshes": [
                {"corners": UNIT, "d": 2},
                {"corners": shifted(1.0, 0.0), "d": 2},
                {"corners": shifted(0.0, 1.0), "d": 2, "tags": {"top": "clamped"}},
            ],
            "material": (1.0, 0.3, "plane-strain"), "eps": 1e-8, "body": (0.0, -1.0), "solve": 1e-8,
        },
        "cantilever2": {
            "meshes": [
                {"corners": UNIT, "d": 2, "tags": {"left": "clamped"}},
                {"corners": shifted(1.0, 0.0), "d": 2, "tractions": {"right": (0.0, 1.0)}},
            ],
            "material": (64.0, 0.0, "plane-stress"), "eps": 1e-12, "body": (0.0, 0.0), "solve": 1e-9,
        },
    }
