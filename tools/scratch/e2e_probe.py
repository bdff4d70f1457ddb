"""Where the config-2 end-to-end time goes: H2D construction, device work,
D2H numpy_cores, per pair (serial) and concurrent total."""
import sys, time
sys.path.insert(0, '.')
import torch
from bench import make_inputs, EPS, PAIRS
from paper_2501_07778_b200 import ttcore as T, _lib
host = {p: make_inputs(*p) for p in PAIRS}
def job(p, tm=None):
    t0 = time.perf_counter(); A = T.TTMatrix(host[p][0]); x = T.TTVector(host[p][1]); torch.cuda.synchronize(); t1 = time.perf_counter()
    z = T.tt_round(T.tt_matvec(A, x), EPS); torch.cuda.synchronize(); t2 = time.perf_counter()
    c = z.numpy_cores(); t3 = time.perf_counter()
    if tm is not None: tm[p] = (round((t1 - t0) * 1e3, 1), round((t2 - t1) * 1e3, 1), round((t3 - t2) * 1e3, 1), round(sum(a.nbytes for a in c) / 1e6, 1))
    return z
for rep in range(3):
    tm = {}
    t0 = time.perf_counter()
    for p in PAIRS: job(p, tm)
    ts = time.perf_counter() - t0
    t0 = time.perf_counter()
    _lib.run_concurrent([(job, p) for p in PAIRS]); torch.cuda.synchronize()
    tc = time.perf_counter() - t0
    print(f"serial {ts*1e3:.1f} ms  concurrent {tc*1e3:.1f} ms")
for p, v in tm.items(): print(p, "h2d ms, compute ms, d2h ms, MB:", v)
