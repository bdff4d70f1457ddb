"""TT serialization and CSV solve reports (the
reference declares both -- a flat container "header (d, mode sizes, ranks) +
cores in row-major order" and the bench_cli CSV columns -- but ships
neither; this module follows the SPEC text).

Container layout (little endian), documented here as the SPEC asks:

    magic   8 bytes  b"QTTB200\\0"
    kind    int32    0 = TTVector, 1 = TTMatrix
    d       int32
    rows    d x int64   row mode sizes
    cols    d x int64   column mode sizes (1 for vectors)
    ranks   (d+1) x int64
    cores   float64, core by core, each C-order (row-major) in the reference
            layout (r, n, r') / (r, n, m, r')

Pure host code (numpy + struct): importable without a GPU; ``load_tt``
builds the device object only when asked to.
"""

from __future__ import annotations

import csv
import io
import struct
from dataclasses import asdict, dataclass, fields

import numpy as np

MAGIC = b"QTTB200\0"

__all__ = ["save_tt", "load_tt", "dump_cores", "parse_cores", "SolveReport", "CSV_COLUMNS", "write_csv",
           "read_csv"]


def dump_cores(cores, is_matrix: bool) -> bytes:
    """Serialize a list of host cores (order 3, or order 4 for matrices)."""
    cores = [np.ascontiguousarray(c, dtype="<f8") for c in cores]
    d = len(cores)
    want = 4 if is_matrix else 3
    if d == 0 or any(c.ndim != want for c in cores):
        raise ValueError("cores must be a non-empty list of order-%d arrays" % want)
    rows = [c.shape[1] for c in cores]
    cols = [c.shape[2] if is_matrix else 1 for c in cores]
    ranks = [c.shape[0] for c in cores] + [cores[-1].shape[-1]]
    for a, b in zip(cores[:-1], cores[1:]):
        if a.shape[-1] != b.shape[0]:
            raise ValueError("adjacent core ranks do not match")
    out = io.BytesIO()
    out.write(MAGIC)
    out.write(struct.pack("<ii", 1 if is_matrix else 0, d))
    out.write(np.asarray(rows, dtype="<i8").tobytes())
    out.write(np.asarray(cols, dtype="<i8").tobytes())
    out.write(np.asarray(ranks, dtype="<i8").tobytes())
    for c in cores:
        out.write(c.tobytes(order="C"))
    return out.getvalue()


def parse_cores(blob: bytes):
    """Inverse of dump_cores: (list of host cores, is_matrix)."""
    if blob[:8] != MAGIC:
        raise ValueError("not a QTTB200 tensor-train container")
    kind, d = struct.unpack_from("<ii", blob, 8)
    if kind not in (0, 1) or d < 1:
        raise ValueError("corrupt header")
    off = 16
    rows = np.frombuffer(blob, dtype="<i8", count=d, offset=off); off += 8 * d
    cols = np.frombuffer(blob, dtype="<i8", count=d, offset=off); off += 8 * d
    ranks = np.frombuffer(blob, dtype="<i8", count=d + 1, offset=off); off += 8 * (d + 1)
    cores = []
    for l in range(d):
        shp = (int(ranks[l]), int(rows[l]), int(cols[l]), int(ranks[l + 1])) if kind else \
              (int(ranks[l]), int(rows[l]), int(ranks[l + 1]))
        n = int(np.prod(shp))
        if off + 8 * n > len(blob):
            raise ValueError("truncated container")
        cores.append(np.frombuffer(blob, dtype="<f8", count=n, offset=off).reshape(shp).copy())
        off += 8 * n
    if off != len(blob):
        raise ValueError("trailing bytes in container")
    return cores, bool(kind)


def save_tt(path, t) -> None:
    """Write a TTVector / TTMatrix (or a plain list of host cores) to ``path``."""
    cores = list(t.cores) if hasattr(t, "cores") else list(t)
    is_matrix = cores[0].ndim == 4
    with open(path, "wb") as f:
        f.write(dump_cores(cores, is_matrix))


def load_tt(path, device: bool = True):
    """Read a container; returns a TTVector / TTMatrix on the GPU, or the
    list of host cores with ``device=False``."""
    with open(path, "rb") as f:
        cores, is_matrix = parse_cores(f.read())
    if not device:
        return cores
    from . import ttcore

    return ttcore.TTMatrix(cores) if is_matrix else ttcore.TTVector(cores)


# ------------------------------------------------------------ CSV reports

CSV_COLUMNS = ("case", "d", "eps", "dofs", "energy_error", "l2_error", "Rd", "Nd", "erank_K", "erank_f",
               "erank_u", "storage_K", "storage_f", "wall_ms", "converged", "drift")


@dataclass(frozen=True)
class SolveReport:
    """One row of the bench CSV."""
    case: str
    d: int
    eps: float
    dofs: int
    energy_error: float
    l2_error: float
    Rd: int
    Nd: int
    erank_K: float
    erank_f: float
    erank_u: float
    storage_K: int
    storage_f: int
    wall_ms: float
    converged: bool
    drift: bool = False


def write_csv(path_or_file, reports) -> None:
    own = isinstance(path_or_file, (str, bytes))
    f = open(path_or_file, "w", newline="") if own else path_or_file
    try:
        w = csv.writer(f)
        w.writerow(CSV_COLUMNS)
        for r in reports:
            row = asdict(r)
            w.writerow([repr(row[c]) if isinstance(row[c], float) else row[c] for c in CSV_COLUMNS])
    finally:
        if own:
            f.close()


def read_csv(path_or_file) -> list:
    own = isinstance(path_or_file, (str, bytes))
    f = open(path_or_file, newline="") if own else path_or_file
    try:
        rd = csv.DictReader(f)
        if tuple(rd.fieldnames or ()) != CSV_COLUMNS:
            raise ValueError("unexpected CSV columns")
        types = {fl.name: fl.type for fl in fields(SolveReport)}
        out = []
        for row in rd:
            kw = {}
            for c in CSV_COLUMNS:
                t = types[c]
                v = row[c]
                if t in ("int", int):
                    kw[c] = int(v)
                elif t in ("float", float):
                    kw[c] = float(v)
                elif t in ("bool", bool):
                    kw[c] = v == "True"
                else:
                    kw[c] = v
            out.append(SolveReport(**kw))
        return out
    finally:
        if own:
            f.close()
