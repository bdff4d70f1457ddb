"""Diagnostic: where does the config-4 forward error against the conforming
splu solution come from -- the assembly tolerance (operator perturbation) or
the AMEn solve?  Assembles at several tolerances, solves at eps = 1e-8.

Usage: python tools/c4_error_probe.py D"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2501_07778_b200 import solver as S
from paper_2501_07778_b200 import ttcore as T
from paper_2501_07778_b200.assembly import assemble_subdomain
from paper_2501_07778_b200.configs import config
from paper_2501_07778_b200.coupling import apply_dirichlet, concat_blocks
from paper_2501_07778_b200.topology import DomainTopology

d = int(sys.argv[1])
c = np.load(f"tests/golden/conforming_c4_d{d}.npz")
uc = T.TTVector([c[f"cores_{k}"] for k in range(len(c["ranks"]) - 1)])
print("conforming ranks", uc.ranks, "compress_err", float(c["compress_err"]), flush=True)


def rel(a, b):
    return T.tt_norm(T.tt_sub(a, b)) / T.tt_norm(b)


def build(eps_asm):
    meshes, mat, body, _ = config(4, d)
    systems = [assemble_subdomain(m, mat, "zorder", eps_asm, body_force=body) for m in meshes]
    topo = DomainTopology.from_subdomains(meshes)
    g = concat_blocks(systems, topo, ordering="zorder", epsilon=eps_asm)
    return apply_dirichlet(g, epsilon=eps_asm)


UP = dict(local_solver="auto", truncation="residual", enrichment_rank=24, local_rtol_factor=1e-3)
for eps_asm, eps_solve in [(1e-8, 1e-8), (1e-8, 1e-10), (1e-10, 1e-8), (1e-12, 1e-8), (1e-12, 1e-10)]:
    t0 = time.perf_counter()
    g = build(eps_asm)
    torch.cuda.synchronize()
    tb = time.perf_counter() - t0
    res_c = S.residual(g.K, uc, g.f)
    t0 = time.perf_counter()
    res = S.solve(g.K, g.f, S.SolverConfig(epsilon=eps_solve, seed=0, max_sweeps=30, stall_sweeps=5, **UP))
    ts = time.perf_counter() - t0
    print(json.dumps({"eps_asm": eps_asm, "eps_solve": eps_solve, "K_max_rank": max(g.K.ranks), "build_s": round(tb, 2),
                      "residual_of_conforming_u": res_c, "solve_s": round(ts, 2), "sweeps": res.sweeps,
                      "residual": res.residual, "max_rank": max(res.u.ranks),
                      "err_vs_conforming": rel(res.u, uc)}), flush=True)
