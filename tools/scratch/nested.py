"""Experiment: nested iteration for the variable-E config-4 AMEn solve.
Solve at level d0, bilinearly interpolate the dense solution to d0+1, TT-SVD
it as the initial guess of the next level (single patch layout Z + 4^d c)."""
import sys, time, json, argparse
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2501_07778_b200.configs import build_system
from paper_2501_07778_b200 import solver as S, ttcore as T
from paper_2501_07778_b200.indexing import zorder_permutation
ap = argparse.ArgumentParser(); ap.add_argument('--d0', type=int, default=7); ap.add_argument('--d1', type=int, default=8)
ap.add_argument('--rho', type=int, default=8); ap.add_argument('--init-eps', type=float, default=1e-10)
ap.add_argument('--config', type=int, default=4); ap.add_argument('--max-sweeps', type=int, default=40)
a = ap.parse_args()
T._CONTRACT_GUARD_BITS = 30
dev = torch.device('cuda')

def grids(u, d):
    perm = torch.from_numpy(zorder_permutation(d)).to(dev)
    n = 2 ** d
    out = []
    for c in range(2):
        g = torch.empty(4 ** d, dtype=torch.float64, device=dev)
        g[perm] = u[c * 4 ** d:(c + 1) * 4 ** d]
        out.append(g.view(n, n))  # [j, i]
    return out

def interp(g, nc, nf):
    x = torch.arange(nf, dtype=torch.float64, device=dev) / (nf - 1) * (nc - 1)
    i0 = torch.clamp(x.floor().long(), max=nc - 2); t = x - i0
    gx = g[:, i0] * (1 - t) + g[:, i0 + 1] * t  # interpolate along i
    return gx[i0, :] * (1 - t)[:, None] + gx[i0 + 1, :] * t[:, None]

def flat(gs, d):
    perm = torch.from_numpy(zorder_permutation(d)).to(dev)
    return torch.cat([g.reshape(-1)[perm] for g in gs])

x0 = None
for d in range(a.d0, a.d1 + 1):
    t0 = time.perf_counter()
    gsys, eps = build_system(a.config, d)
    t1 = time.perf_counter()
    out = S.solve(gsys.K, gsys.f, S.SolverConfig(epsilon=eps, seed=0, max_sweeps=a.max_sweeps, truncation='residual',
                                                 enrichment_rank=a.rho), x0=x0)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(json.dumps({'d': d, 'build_s': t1 - t0, 'solve_s': t2 - t1, 'sweeps': out.sweeps, 'res': out.residual,
                      'conv': out.converged, 'ranks': out.u.ranks, 'x0_ranks': None if x0 is None else x0.ranks,
                      'res_hist': out.residual_history, 'rank_hist': out.rank_history}), flush=True)
    if d == a.d1: break
    u = T.tt_contract_device(out.u)
    gs = [interp(g, 2 ** d, 2 ** (d + 1)) for g in grids(u, d)]
    x0 = T.tt_decompose(flat(gs, d + 1), a.init_eps)
