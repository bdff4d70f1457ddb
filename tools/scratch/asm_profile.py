"""Phase timing of the variable-E config-4 assembly (synchronising timers
around the TT primitives assemble_subdomain calls)."""
import sys, time, collections
sys.path.insert(0, '.')
import torch
from paper_2501_07778_b200 import assembly as A, ttcore as T, configs
d = int(sys.argv[1]) if len(sys.argv) > 1 else 10
acc = collections.defaultdict(float); cnt = collections.Counter()
def wrap(mod, name):
    f = getattr(mod, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter(); r = f(*a, **k); torch.cuda.synchronize()
        acc[name] += time.perf_counter() - t; cnt[name] += 1; return r
    setattr(mod, name, g)
for n in ("tt_decompose", "tt_diag", "tt_matmat", "tt_add", "tt_round", "value_grids", "tt_matvec", "tt_scale"):
    if hasattr(A, n): wrap(A, n)
meshes, mat, body, eps = configs.config(int(sys.argv[2]) if len(sys.argv) > 2 else 4, d)
torch.cuda.synchronize(); t0 = time.perf_counter()
s = A.assemble_subdomain(meshes[0], mat, "zorder", eps, body_force=body, cache=False)
torch.cuda.synchronize(); print("total", time.perf_counter() - t0)
for k, v in sorted(acc.items(), key=lambda x: -x[1]): print(f"{k:14s} {v:8.3f} s  x{cnt[k]}")
print("kxx ranks", s.kxx.ranks)
