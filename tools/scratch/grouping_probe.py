"""Concurrent config-2 step with the 9 pairs grouped into fewer chains (less SM contention?)."""
import sys, time; sys.path.insert(0, ".")
import torch
from bench import make_inputs, EPS, PAIRS
from paper_2501_07778_b200 import ttcore as T, _lib
host = {p: make_inputs(*p) for p in PAIRS}
res = {p: (T.TTMatrix(host[p][0]), T.TTVector(host[p][1])) for p in PAIRS}
def chain(ps):
    out = None
    for p in ps:
        A, x = res[p]
        out = T.tt_round(T.tt_matvec(A, x), EPS)
    return out
GROUPINGS = {
    "9 chains": [[p] for p in sorted(PAIRS, key=lambda p: -p[0] * p[1])],
    "4 chains": [[(16, 128)], [(8, 128), (16, 64)], [(4, 128), (8, 64), (4, 16), (8, 16)], [(4, 64), (16, 16)]],
    "3 chains": [[(16, 128)], [(8, 128), (16, 64)], [(4, 128), (8, 64), (4, 64), (16, 16), (8, 16), (4, 16)]],
    "5 chains": [[(16, 128)], [(8, 128)], [(16, 64)], [(4, 128), (8, 64), (4, 16)], [(4, 64), (16, 16), (8, 16)]],
    "6 chains": [[(16, 128)], [(8, 128)], [(16, 64)], [(4, 128), (4, 16)], [(8, 64), (8, 16)], [(4, 64), (16, 16)]],
}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
import os
ORDER = ["9 chains", "6 chains", "9 chains", "6 chains", "7 chains", "9 chains", "6 chains"] if os.environ.get("AB") else list(GROUPINGS)
GROUPINGS["7 chains"] = [[(16, 128)], [(8, 128)], [(16, 64)], [(4, 128)], [(8, 64)], [(4, 64), (4, 16)], [(16, 16), (8, 16)]]
for name in ORDER:
    groups = GROUPINGS[name]
    for _ in range(2): _lib.run_concurrent([(chain, g) for g in groups])
    ts = []
    for _ in range(5):
        flush.zero_(); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); _lib.run_concurrent([(chain, g) for g in groups]); e1.record(); torch.cuda.synchronize()
        ts.append(round(e0.elapsed_time(e1), 2))
    print(name, ts, flush=True)
