"""Build (assembly + coupling + Dirichlet) time of a config, second run in-process."""
import sys, time, json
sys.path.insert(0, '.')
import torch
from paper_2501_07778_b200.configs import build_system
idx = int(sys.argv[1]); d = int(sys.argv[2]) if len(sys.argv) > 2 else None
from paper_2501_07778_b200 import assembly as _A
for rep in range(3):
    _A._assembly_cache.clear()
    tm = {}
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g, eps = build_system(idx, d, tm)
    torch.cuda.synchronize()
    print(rep, round(time.perf_counter() - t0, 3), {k: round(v, 3) for k, v in tm.items()}, max(g.K.ranks), flush=True)
