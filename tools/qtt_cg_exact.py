"""Diagnostic: exact solution of the coupled QTT system (penalty coupling,
coupling.py:333-485) by Jacobi-preconditioned CG on the dense vector with the
device TT-matrix apply, to separate the AMEn error from the difference
between the penalty-coupled QTT system and the merged-node conforming FEM.

Usage: python tools/qtt_cg_exact.py CONFIG D"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2501_07778_b200 import solver as S
from paper_2501_07778_b200 import ttcore as T
from paper_2501_07778_b200.configs import build_system

idx, d = int(sys.argv[1]), int(sys.argv[2])
gsys, eps = build_system(idx, d)
K, f = gsys.K, gsys.f
fd = T.tt_contract_device(f)
# diagonal of K: cores C[:, i, i, :]
diag_cores = [c[:, [0, 1], [0, 1], :].contiguous() for c in K.device_cores]
dg = T.tt_contract_device(T.TTVector(diag_cores))
dinv = 1.0 / dg
x = torch.zeros_like(fd)
r = fd.clone()
z = dinv * r
p = z.clone()
rz = torch.dot(r, z)
nb = float(torch.linalg.vector_norm(fd))
t0 = time.perf_counter()
hist = []
for it in range(200000):
    Ap = S.apply_tt_matrix(K, p)
    a = rz / torch.dot(p, Ap)
    x += a * p
    r -= a * Ap
    if it % 500 == 0:
        rel = float(torch.linalg.vector_norm(r)) / nb
        hist.append((it, rel))
        if rel < 1e-15 or time.perf_counter() - t0 > 600:
            break
    z = dinv * r
    rz2 = torch.dot(r, z)
    p = z + (rz2 / rz) * p
    rz = rz2
true_res = float(torch.linalg.vector_norm(S.apply_tt_matrix(K, x) - fd)) / nb
out = {"config": idx, "d": d, "cg_iters": it + 1, "cg_s": time.perf_counter() - t0, "cg_true_res": true_res,
       "hist_tail": hist[-4:]}
c = np.load(f"tests/golden/conforming_c{idx}_d{d}.npz")
uc = T.tt_contract_device(T.TTVector([c[f"cores_{k}"] for k in range(len(c["ranks"]) - 1)]))
nuc = float(torch.linalg.vector_norm(uc))
out["qtt_exact_vs_conforming"] = float(torch.linalg.vector_norm(x - uc)) / nuc
S._DENSE_RESIDUAL_BITS = 23
res = S.solve(K, f, S.SolverConfig(epsilon=eps, seed=0, local_solver="auto", truncation="residual",
                                   enrichment_rank=24, local_rtol_factor=1e-3, max_sweeps=30, stall_sweeps=4))
ua = T.tt_contract_device(res.u)
out["amen_vs_qtt_exact"] = float(torch.linalg.vector_norm(ua - x) / torch.linalg.vector_norm(x))
out["amen_vs_conforming"] = float(torch.linalg.vector_norm(ua - uc)) / nuc
out["amen_residual"] = res.residual
out["amen_sweeps"] = res.sweeps
print(json.dumps(out), flush=True)
