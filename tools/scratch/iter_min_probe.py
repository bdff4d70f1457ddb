"""GMRES / dense-LU crossover (solver._ITERATIVE_MIN_DIM) on config 4, both assembly tolerances."""
import sys, time, json
sys.path.insert(0, '.')
import torch
from paper_2501_07778_b200 import solver as S
from paper_2501_07778_b200.configs import build_system
UP = dict(local_solver="auto", truncation="residual", enrichment_rank=24, local_rtol_factor=1e-3)
for asm in (None, 1e-12):
    gsys, eps = build_system(4, 10, assembly_eps=asm)
    for m in (8192, 4096, 8192, 4096, 2048):
        S._ITERATIVE_MIN_DIM = m
        torch.cuda.synchronize(); t0 = time.perf_counter()
        res = S.solve(gsys.K, gsys.f, S.SolverConfig(epsilon=eps, seed=0, **UP))
        torch.cuda.synchronize()
        print(json.dumps({"asm": asm, "iter_min": m, "solve_s": round(time.perf_counter() - t0, 2), "sweeps": res.sweeps,
                          "residual": res.residual, "max_rank": max(res.u.ranks)}), flush=True)
