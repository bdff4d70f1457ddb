import sys; sys.path.insert(0, ".")
import numpy as np
from paper_2501_07778_b200 import solver as S, ttcore as T
from paper_2501_07778_b200.configs import build_system
gsys, eps = build_system(5, 8)
CONFIG5 = dict(local_solver="auto", truncation="residual", enrichment_rank=24, local_rtol_factor=1e-3, trunc_factor=0.05)
res = S.solve(gsys.K, gsys.f, S.SolverConfig(epsilon=eps, seed=0, max_sweeps=25, stall_sweeps=4, refine_steps=2, **CONFIG5))
c = np.load("tests/golden/conforming_c5_d8.npz")
uc = T.TTVector([c[f"cores_{k}"] for k in range(len(c["ranks"]) - 1)])
print("converged", res.converged, "residual", res.residual, "sweeps", res.sweeps, "err", T.tt_norm(T.tt_sub(res.u, uc)) / T.tt_norm(uc), "hist", res.residual_history[-3:])
