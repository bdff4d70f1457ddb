import sys, time; sys.path.insert(0, ".")
import torch
from bench import make_inputs, EPS, PAIRS
from paper_2501_07778_b200 import ttcore as T
res = {p: (T.TTMatrix(make_inputs(*p)[0]), T.TTVector(make_inputs(*p)[1])) for p in PAIRS}
for rep in range(3):
    tot_dev = 0.0; tot_wall = 0.0; rows = []
    for p in PAIRS:
        A, x = res[p]
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e2 = torch.cuda.Event(enable_timing=True)
        e0.record(); y = T.tt_matvec(A, x); e1.record(); z = T.tt_round(y, EPS); e2.record(); torch.cuda.synchronize()
        w1 = time.perf_counter()
        rows.append((p, round(e0.elapsed_time(e1), 2), round(e1.elapsed_time(e2), 2), round((w1 - w0) * 1e3, 2)))
        tot_dev += e0.elapsed_time(e2); tot_wall += (w1 - w0) * 1e3
    print(rep, "device ms", round(tot_dev, 1), "wall ms", round(tot_wall, 1))
for r in rows: print(r)
