"""Dump a few mid-size AMEn local systems of the config-4 variable-E solve
(d=8 reproduces the same failing shapes quickly) for offline preconditioner
experiments: phi_l, A core, phi_r, rhs, x_cur -> gpurun_out/local_*.npz."""
import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2501_07778_b200.configs import build_system
from paper_2501_07778_b200 import solver as S
d = int(sys.argv[1]) if len(sys.argv) > 1 else 10
want = int(sys.argv[2]) if len(sys.argv) > 2 else 4
os.makedirs("gpurun_out", exist_ok=True)
gsys, eps = build_system(4, d, {})
cnt = [0]
def hook(phi_l, a_p, phi_r, rhs, x_cur, sol):
    rl, n, rr = rhs.shape
    dim = rl * n * rr
    if cnt[0] >= want or not (8000 < dim < 20000):
        return
    ra, rb = a_p["ra"], a_p["rb"]
    its = []
    _, ok, it = S._gmres(phi_l, a_p, phi_r, rhs, x_cur if x_cur is not None else torch.zeros_like(rhs), 2e-10, maxit=400)
    if ok and it < 150:
        return
    np.savez(f"gpurun_out/local_{cnt[0]}.npz", phi_l=phi_l.cpu().numpy(), a=a_p["a_ijb"].cpu().numpy().reshape(ra, n, n, rb),
             phi_r=phi_r.cpu().numpy(), rhs=rhs.cpu().numpy(), x_cur=x_cur.cpu().numpy() if x_cur is not None else np.zeros(rhs.shape),
             its=it, ok=ok)
    print("dumped", cnt[0], (rl, n, rr, ra, rb), "its", it, "ok", ok, flush=True)
    cnt[0] += 1
S._LOCAL_HOOK = hook
cfg = S.SolverConfig(epsilon=eps, seed=0, local_solver="auto", truncation="residual", enrichment_rank=16, max_sweeps=8)
S.solve(gsys.K, gsys.f, cfg)
