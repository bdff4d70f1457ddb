import sys, time; sys.path.insert(0, ".")
import torch
from bench import make_inputs, EPS, PAIRS
from paper_2501_07778_b200 import ttcore as T, _lib
host = {p: make_inputs(*p) for p in PAIRS}
res = {p: (T.TTMatrix(host[p][0]), T.TTVector(host[p][1])) for p in PAIRS}
def pair_job(p):
    A, x = res[p]
    return T.tt_round(T.tt_matvec(A, x), EPS)
def serial(tag):
    rows = []
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for p in PAIRS:
        t1 = time.perf_counter(); z = pair_job(p); torch.cuda.synchronize(); rows.append(round((time.perf_counter() - t1) * 1e3, 2))
    print(tag, round((time.perf_counter() - t0) * 1e3, 1), rows, flush=True)
order = sorted(PAIRS, key=lambda p: -p[0] * p[1])
serial("cold"); serial("warm")
_lib.run_concurrent([(pair_job, p) for p in order]); torch.cuda.synchronize()
serial("after-1-concurrent")
torch.cuda.empty_cache(); serial("after-empty_cache")
_lib.run_concurrent([(pair_job, p) for p in order]); torch.cuda.synchronize()
serial("after-concurrent-again")
_lib.release_cached(); serial("after-release_cached"); serial("again")
