import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2501_07778_b200 import solver as S, ttcore as T
from paper_2501_07778_b200.configs import build_system
d = int(sys.argv[1])
S._DENSE_RESIDUAL_BITS = 23
S._TRACE = True
gsys, eps = build_system(5, d)
c = np.load(f"tests/golden/conforming_c5_d{d}.npz")
uc = T.TTVector([c[f"cores_{k}"] for k in range(len(c["ranks"]) - 1)])
for rs, rt in ((2, 1e-2), (1, 1e-3)):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = S.solve(gsys.K, gsys.f, S.SolverConfig(epsilon=eps, seed=0, local_solver="auto", truncation="residual",
                  enrichment_rank=24, local_rtol_factor=1e-3, trunc_factor=0.05, stall_sweeps=4, max_sweeps=30,
                  refine_steps=rs, refine_tol=rt))
    torch.cuda.synchronize()
    print(json.dumps({"refine_steps": rs, "refine_tol": rt, "solve_s": round(time.perf_counter() - t0, 2), "sweeps": res.sweeps,
                      "residual": res.residual, "max_rank": max(res.u.ranks),
                      "err_vs_conforming": T.tt_norm(T.tt_sub(res.u, uc)) / T.tt_norm(uc)}), flush=True)
