"""Dense residual apply: split left/right contraction vs the dense chain
over a materialised u (config-4 operator, random u of rank r)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2501_07778_b200.configs import build_system
from paper_2501_07778_b200 import solver as S, ttcore as T
gsys, eps = build_system(4, 10, {})
K = gsys.K
rng = np.random.default_rng(0)
d = K.d
for r in (64, 128, 271):
    rk = [1] + [min(r, 2 ** min(k, d - k)) for k in range(1, d)] + [1]
    u = T.TTVector([rng.standard_normal((rk[k], 2, rk[k + 1])) / np.sqrt(rk[k]) for k in range(d)])
    for name, fn in (("split", lambda: S._apply_tt_to_tt(K, u)), ("chain", lambda: S.apply_tt_matrix(K, T.tt_contract_device(u)))):
        fn(); torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(3): y = fn()
        torch.cuda.synchronize(); print(f"r={r} {name}: {(time.perf_counter() - t) / 3 * 1e3:.1f} ms", flush=True)
