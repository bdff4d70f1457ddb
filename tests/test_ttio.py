"""TT container and CSV report round trips: host-only."""
import io
import math

import numpy as np
import pytest

from paper_2501_07778_b200 import ttio


def _cores(rng, shapes):
    return [rng.standard_normal(s) for s in shapes]


def test_container_round_trip_vector_and_matrix(tmp_path):
    rng = np.random.default_rng(0)
    vec = _cores(rng, [(1, 2, 3), (3, 2, 5), (5, 3, 1)])
    mat = _cores(rng, [(1, 2, 2, 4), (4, 2, 2, 1)])
    for cores, is_matrix in ((vec, False), (mat, True)):
        blob = ttio.dump_cores(cores, is_matrix)
        back, kind = ttio.parse_cores(blob)
        assert kind == is_matrix
        assert all(np.array_equal(a, b) for a, b in zip(cores, back))
        p = tmp_path / "t.qtt"
        ttio.save_tt(p, cores)
        assert all(np.array_equal(a, b) for a, b in zip(cores, ttio.load_tt(p, device=False)))


def test_container_rejects_corruption():
    rng = np.random.default_rng(1)
    blob = ttio.dump_cores(_cores(rng, [(1, 2, 2), (2, 2, 1)]), False)
    with pytest.raises(ValueError):
        ttio.parse_cores(b"XXXXXXXX" + blob[8:])
    with pytest.raises(ValueError):
        ttio.parse_cores(blob[:-8])
    with pytest.raises(ValueError):
        ttio.parse_cores(blob + b"\0" * 8)
    with pytest.raises(ValueError):
        ttio.dump_cores(_cores(rng, [(1, 2, 2), (3, 2, 1)]), False)


def test_csv_round_trip_is_exact():
    rows = [
        ttio.SolveReport("config1", 5, 1e-8, 2048, math.nan, 1.2345678901234567e-10, 32, 4711, 40.25, 2.5, 19.75,
                         123456, 99, 371.25, True),
        ttio.SolveReport("config5", 10, 1e-8, 6291456, math.nan, math.nan, 109, 10**7, 80.0, 3.0, 60.5,
                         10**8, 1000, 10246.5, False, True),
    ]
    f = io.StringIO()
    ttio.write_csv(f, rows)
    assert f.getvalue().splitlines()[0] == ",".join(ttio.CSV_COLUMNS)
    f.seek(0)
    back = ttio.read_csv(f)
    for a, b in zip(rows, back):
        for c in ttio.CSV_COLUMNS:
            x, y = getattr(a, c), getattr(b, c)
            assert (x == y) or (isinstance(x, float) and math.isnan(x) and math.isnan(y)), c


def test_cli_argument_checks():
    from paper_2501_07778_b200 import cli

    with pytest.raises(SystemExit):
        cli.main(["run", "--case", "config1", "--d", "3", "4"])
    with pytest.raises(SystemExit):
        cli.main(["run", "--case", "nope", "--d", "3"])
    with pytest.raises(SystemExit):
        cli.main(["sweep", "--case", "config1", "--d", "1"])
