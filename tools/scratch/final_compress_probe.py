"""Cost split of _final_compress on the converged config-4 iterate:
tt_round (R->L + L->R) vs tt_norm (R->L only) vs residual."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2501_07778_b200.configs import build_system
from paper_2501_07778_b200 import solver as S, ttcore as T
gsys, eps = build_system(4, 10, {})
out = S.solve(gsys.K, gsys.f, S.SolverConfig(epsilon=eps, seed=0, local_solver="auto", truncation="residual",
                                             enrichment_rank=24, local_rtol_factor=1e-3))
u = out.u
def tm(f, n=3):
    f(); torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(n): r = f()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / n * 1e3, r
for fac in (0.5, 0.003):
    ms, c = tm(lambda: T.tt_round(u, fac * eps))
    print(f"round {fac}: {ms:.1f} ms ranks max {max(c.ranks)}")
ms, _ = tm(lambda: T.tt_norm(u)); print(f"R->L only (tt_norm): {ms:.1f} ms")
ms, _ = tm(lambda: S.residual(gsys.K, u, gsys.f)); print(f"residual: {ms:.1f} ms")
t = time.perf_counter(); S._final_compress(gsys.K, gsys.f, u, out.residual, eps); torch.cuda.synchronize()
print(f"_final_compress: {(time.perf_counter() - t) * 1e3:.1f} ms; u ranks max {max(u.ranks)}")
