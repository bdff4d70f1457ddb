"""Diagnostic: is the config-5 AMEn plateau a solver stall or the FP64 floor
of the residual itself?  Builds config 5 at level d, runs AMEn for a few
sweeps, then evaluates

* the residual of the iterate by two contraction orders (half-split GEMM
  meeting vs dense chain over the materialised u),
* the residual of the CONFORMING splu solution scattered into the QTT layout
  (tests/golden/conforming_c5_d{d}.npz), which is accurate to ~1e-10 in u,
* the forward error of the iterate against that conforming solution,
* kappa_u = ||K||_2 ||u|| / ||f|| (power iteration on the dense apply).

Usage: python tools/residual_floor.py D SWEEPS
"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2501_07778_b200 import solver as S
from paper_2501_07778_b200 import ttcore as T
from paper_2501_07778_b200.configs import build_system

d = int(sys.argv[1])
sweeps = int(sys.argv[2])
cfg_idx = int(sys.argv[3]) if len(sys.argv) > 3 else 5
tf = float(sys.argv[4]) if len(sys.argv) > 4 else 0.5
stall = int(sys.argv[5]) if len(sys.argv) > 5 else 0
rtf = float(sys.argv[6]) if len(sys.argv) > 6 else 1e-3
S._DENSE_RESIDUAL_BITS = 23
gsys, eps = build_system(cfg_idx, d)
K, f = gsys.K, gsys.f
out = {"d": d, "K_ranks": K.ranks}
res = S.solve(K, f, S.SolverConfig(epsilon=eps, seed=0, local_solver="auto", truncation="residual",
                                   enrichment_rank=24, local_rtol_factor=rtf, max_sweeps=sweeps,
                                   trunc_factor=tf, stall_sweeps=stall))
out.update(tf=tf, rtf=rtf, sweeps=res.sweeps, solve_s=res.wall_time, u_ranks=max(res.u.ranks))
u = res.u
out["res_hist"] = [float(x) for x in res.residual_history]
fd = T.tt_contract_device(f)
nf = float(torch.linalg.vector_norm(fd))
r1 = float(torch.linalg.vector_norm(S._apply_tt_to_tt(K, u) - fd)) / nf
ud = T.tt_contract_device(u)
r2 = float(torch.linalg.vector_norm(S.apply_tt_matrix(K, ud) - fd)) / nf
out.update(res_split=r1, res_chain=r2)
# perturb u by 1e-13 relative noise: how much does the evaluated residual move?
g = torch.Generator(device="cuda").manual_seed(1)
up = ud * (1 + 1e-13 * torch.randn(ud.shape, generator=g, device="cuda", dtype=torch.float64))
out["res_chain_perturbed_1e-13"] = float(torch.linalg.vector_norm(S.apply_tt_matrix(K, up) - fd)) / nf
# ||K||_2 by power iteration
x = torch.randn(ud.shape, generator=g, device="cuda", dtype=torch.float64)
for _ in range(30 if d < 10 else 8):
    x = S.apply_tt_matrix(K, x)
    x /= torch.linalg.vector_norm(x)
lam = float(torch.linalg.vector_norm(S.apply_tt_matrix(K, x)))
nu = float(torch.linalg.vector_norm(ud))
out.update(K_norm2=lam, u_norm=nu, f_norm=nf, kappa_u=lam * nu / nf)
try:
    c = np.load(f"tests/golden/conforming_c{cfg_idx}_d{d}.npz")
    uc = T.TTVector([c[f"cores_{k}"] for k in range(len(c["ranks"]) - 1)])
    ucd = T.tt_contract_device(uc)
    out["conf_err"] = float(torch.linalg.vector_norm(ud - ucd) / torch.linalg.vector_norm(ucd))
    out["res_of_conforming_split"] = float(torch.linalg.vector_norm(S._apply_tt_to_tt(K, uc) - fd)) / nf
    out["res_of_conforming_chain"] = float(torch.linalg.vector_norm(S.apply_tt_matrix(K, ucd) - fd)) / nf
except FileNotFoundError:
    pass
print(json.dumps(out), flush=True)
