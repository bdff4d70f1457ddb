import sys, time, json, argparse
sys.path.insert(0, '.')
import torch
from paper_2501_07778_b200.configs import build_system
from paper_2501_07778_b200 import solver as S
ap = argparse.ArgumentParser(); ap.add_argument('--config', type=int, default=1); ap.add_argument('--d', type=int, default=None)
ap.add_argument('--max-sweeps', type=int, default=40); ap.add_argument('--no-solve', action='store_true'); ap.add_argument('--dense-bits', type=int, default=22)
ap.add_argument('--trunc', default='reference'); ap.add_argument('--rho', type=int, default=4); ap.add_argument('--local', default='direct'); ap.add_argument('--rtol-factor', type=float, default=0.0); ap.add_argument('--iter-min', type=int, default=None); ap.add_argument('--trunc-factor', type=float, default=0.5)
a = ap.parse_args()
S._DENSE_RESIDUAL_BITS = a.dense_bits
if a.iter_min is not None: S._ITERATIVE_MIN_DIM = a.iter_min
import os
if os.environ.get('QTT_SOLVER_PROFILE'): S.PROFILE = {}
tm = {}
t0 = time.perf_counter()
gsys, eps = build_system(a.config, a.d, tm)
tm['K_ranks'] = gsys.K.ranks; tm['f_ranks'] = gsys.f.ranks
print(json.dumps(tm), flush=True)
t1 = time.perf_counter()
if a.no_solve: sys.exit(0)
out = S.solve(gsys.K, gsys.f, S.SolverConfig(epsilon=eps, seed=0, local_solver=a.local, max_sweeps=a.max_sweeps, truncation=a.trunc, enrichment_rank=a.rho, local_rtol_factor=a.rtol_factor, trunc_factor=a.trunc_factor))
torch.cuda.synchronize()
t2 = time.perf_counter()
calls = (S.PROFILE or {}).pop('calls', [])
if calls:
    import collections
    agg = collections.defaultdict(lambda: [0, 0, 0.0, 0])
    for kind, rl, ra, rr, its, ok, t in calls:
        key = (kind, (rl * 2 * rr) // 10000)
        agg[key][0] += 1; agg[key][1] += its; agg[key][2] += t; agg[key][3] += (not ok)
    for k in sorted(agg): print('calls', k[0], f'dim~{k[1]*10}k', 'n', agg[k][0], 'its/dim', agg[k][1], 't %.3f' % agg[k][2], 'fail', agg[k][3])
    fails = [c for c in calls if not c[5]]
    print('failed gmres:', fails[:30])
print(json.dumps({'config': a.config, 'd': a.d, 'solve_s': t2 - t1, 'total_s': t2 - t0, 'sweeps': out.sweeps,
                  'residual': out.residual, 'converged': out.converged, 'u_ranks': out.u.ranks,
                  'res_hist': out.residual_history, 'rank_hist': out.rank_history, 'profile': S.PROFILE}), flush=True)
