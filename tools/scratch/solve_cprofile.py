"""cProfile of the config-4 variable-E d=10 solve (wall-clock attribution of
host time, including synchronising calls)."""
import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import torch
from paper_2501_07778_b200.configs import build_system
from paper_2501_07778_b200 import solver as S
d = int(sys.argv[1]) if len(sys.argv) > 1 else 10
gsys, eps = build_system(4, d, {})
torch.cuda.synchronize()
cfg = S.SolverConfig(epsilon=eps, seed=0, local_solver="auto", truncation="residual", enrichment_rank=24, local_rtol_factor=1e-3)
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
out = S.solve(gsys.K, gsys.f, cfg)
torch.cuda.synchronize()
pr.disable()
print("solve", time.perf_counter() - t, out.sweeps)
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(22)
st.sort_stats("cumulative").print_stats(30)
