"""Time the three roundings of apply_dirichlet (config 4, d=10)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2501_07778_b200 import configs, coupling as C, ttcore as T
tm = {}
orig = C.apply_dirichlet
got = {}
def capture(system, *a, **k):
    got['sys'] = system
    return orig(system, *a, **k)
C.apply_dirichlet = capture
gsys, eps = configs.build_system(4, int(sys.argv[1]) if len(sys.argv) > 1 else 10, tm)
system = got.get('sys')
if system is None:
    print("could not capture the global system"); sys.exit(0)
def t(f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize(); return r, time.perf_counter() - t0
dmask = T.tt_diag(system.mask)
dkd, t1 = t(lambda: T.tt_matmat(dmask, T.tt_matmat(system.K, dmask)))
torch.cuda.nvtx.range_push("dkd")
k1, t2 = t(lambda: T.tt_round(dkd, eps))
torch.cuda.nvtx.range_pop()
ones = T.TTVector([np.ones((1, 2, 1))] * system.mask.d)
comp = T.tt_sub(ones, system.mask)
k2, t3 = t(lambda: T.tt_round(T.tt_add(k1, T.tt_scale(T.tt_diag(comp), system.gamma)), eps))
f2, t4 = t(lambda: T.tt_round(T.tt_hadamard(system.mask, system.f), eps))
print(f"matmats {t1:.3f}s round(DKD) {t2:.3f}s [rank {max(dkd.ranks)} -> {max(k1.ranks)}] round(+gamma) {t3:.3f}s round(f) {t4:.3f}s; eps {eps}")
