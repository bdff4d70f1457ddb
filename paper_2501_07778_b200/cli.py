"""Command-line front end (SPEC.md:549-607 ``bench_cli``; declared by the
reference's pyproject but not shipped there): runs the BASELINE geometries
through the device pipeline and emits the SPEC's CSV rows.

    python -m paper_2501_07778_b200.cli run   --case config4 --d 8 --eps 1e-8 --out row.csv
    python -m paper_2501_07778_b200.cli sweep --case config1 --d 3 4 5 --eps 1e-6 1e-8 --out sweep.csv
    python -m paper_2501_07778_b200.cli report sweep.csv
    python -m paper_2501_07778_b200.cli verify --case config5 --d 4

Cases are the BASELINE.json geometries (config1, config4, config4_constE,
config5).  ``l2_error`` is the relative error against the committed
conforming ground truth (tests/golden/conforming_c*_d*.npz) when one exists
for (case, d), else nan; ``energy_error`` needs the reference's conforming
oracle (out of scope) and is nan.  ``--save-u PATH`` snapshots
the solution in the ttio container."""

from __future__ import annotations

import argparse
import math
import os
import sys
import time

from .ttio import SolveReport, read_csv, save_tt, write_csv

CASES = {"config1": 1, "config4": 4, "config4_constE": 40, "config5": 5}
_UPGRADED = dict(local_solver="auto", truncation="residual", enrichment_rank=24, local_rtol_factor=1e-3)
SOLVER = {
    "config1": dict(local_solver="direct"),
    "config4_constE": dict(local_solver="direct"),
    "config4": _UPGRADED,
    "config5": dict(_UPGRADED, trunc_factor=0.05, stall_sweeps=4, max_sweeps=30, refine_steps=1),
}


def run_case(case: str, d: int, eps: float, seed: int = 0, save_u: str | None = None) -> SolveReport:
    """Partition -> assemble -> couple -> mask -> solve -> report."""
    import numpy as np
    import torch

    from . import solver as S
    from . import ttcore as T
    from .assembly import assemble_subdomain
    from .configs import config
    from .coupling import apply_dirichlet, concat_blocks
    from .topology import DomainTopology

    idx = CASES[case]
    meshes, mat, body, _ = config(idx, d)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    systems = [assemble_subdomain(m, mat, "zorder", eps, body_force=body) for m in meshes]
    gsys = concat_blocks(systems, DomainTopology.from_subdomains(meshes), ordering="zorder", epsilon=eps)
    gsys = apply_dirichlet(gsys, epsilon=eps)
    saved = S._DENSE_RESIDUAL_BITS
    if idx == 5:
        S._DENSE_RESIDUAL_BITS = 23
    try:
        res = S.solve(gsys.K, gsys.f, S.SolverConfig(epsilon=eps, seed=seed, **SOLVER[case]))
    finally:
        S._DENSE_RESIDUAL_BITS = saved
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - t0) * 1e3
    l2 = math.nan
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    fx = os.path.join(root, "tests", "golden", f"conforming_c{idx}_d{d}.npz")
    if os.path.exists(fx):
        c = np.load(fx)
        uc = T.TTVector([c[f"cores_{k}"] for k in range(len(c["ranks"]) - 1)])
        l2 = float(T.tt_norm(T.tt_sub(res.u, uc)) / T.tt_norm(uc))
    pk, pf, pu = T.rank_profile(gsys.K), T.rank_profile(gsys.f), T.rank_profile(res.u)
    if save_u:
        save_tt(save_u, res.u)
    q = len(meshes)
    return SolveReport(case=case, d=d, eps=eps, dofs=2 * q * 4**d, energy_error=math.nan, l2_error=l2,
                       Rd=pu.max_rank, Nd=pu.param_count, erank_K=pk.effective_rank,
                       erank_f=pf.effective_rank, erank_u=pu.effective_rank, storage_K=pk.storage_count,
                       storage_f=pf.storage_count, wall_ms=wall_ms, converged=bool(res.converged))


def verify_case(case: str, d: int, eps: float = 1e-8) -> list:
    """SPEC.md:579-586 ``verify`` (d <= 4): dense-equality and
    conforming-equivalence properties of the device pipeline.  Returns a list
    of (property, value, bound, ok)."""
    import numpy as np

    from . import solver as S
    from . import ttcore as T
    from .configs import build_system

    if d > 4:
        raise ValueError("verify needs d <= 4 (dense comparisons)")
    idx = CASES[case]
    gsys, _ = build_system(idx, d)
    res = S.solve(gsys.K, gsys.f, S.SolverConfig(epsilon=eps, seed=0, local_solver="direct"))
    Kd = T.tt_contract(gsys.K)
    fd = T.tt_contract(gsys.f)
    ud = T.tt_contract(res.u)
    checks = []
    if idx != 5:  # the penalty-coupled multi-patch operator is not symmetric (coupling.py:333-485)
        sym = float(np.abs(Kd - Kd.T).max() / np.abs(Kd).max())
        checks.append(("K symmetric (dense)", sym, 1e-10, sym <= 1e-10))
    r_dense = float(np.linalg.norm(Kd @ ud - fd) / np.linalg.norm(fd))
    checks.append(("dense residual ||K u - f|| / ||f||", r_dense, eps, r_dense <= eps))
    u_exact = np.linalg.solve(Kd, fd)
    e_dense = float(np.linalg.norm(ud - u_exact) / np.linalg.norm(u_exact))
    bound = 10 * eps * float(np.linalg.cond(Kd))
    checks.append(("u vs dense solve", e_dense, bound, e_dense <= bound))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    fx = os.path.join(root, "tests", "golden", f"conforming_c{idx}_d{d}.npz")
    if os.path.exists(fx):
        c = np.load(fx)
        uc = T.tt_contract(T.TTVector([c[f"cores_{k}"] for k in range(len(c["ranks"]) - 1)]))
        e_conf = float(np.linalg.norm(ud - uc) / np.linalg.norm(uc))
        checks.append(("u vs conforming FEM (splu fixture)", e_conf, 1e-6, e_conf <= 1e-6))
    return checks


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2501_07778_b200.cli", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("run", "sweep"):
        p = sub.add_parser(name)
        p.add_argument("--case", choices=sorted(CASES), required=True)
        p.add_argument("--d", type=int, nargs="+", required=True)
        p.add_argument("--eps", type=float, nargs="+", default=[1e-8])
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--out", default="-")
        p.add_argument("--save-u", default=None)
    p = sub.add_parser("report")
    p.add_argument("csv")
    p = sub.add_parser("verify")
    p.add_argument("--case", choices=sorted(CASES), required=True)
    p.add_argument("--d", type=int, required=True)
    a = ap.parse_args(argv)
    if a.cmd == "verify":
        if not 2 <= a.d <= 4:
            ap.error("verify takes d in [2, 4]")
        checks = verify_case(a.case, a.d)
        for name, val, bound, ok in checks:
            print(f"{'pass' if ok else 'FAIL'}  {name}: {val:.3e} (bound {bound:.1e})")
        return 0 if all(c[3] for c in checks) else 1
    if a.cmd == "report":
        for r in read_csv(a.csv):
            print(f"{r.case:>16} d={r.d:<2} eps={r.eps:g} dofs={r.dofs} R_d={r.Rd} N_d={r.Nd} "
                  f"erank_u={r.erank_u:.1f} l2={r.l2_error:.2e} wall={r.wall_ms:.0f} ms converged={r.converged}")
        return 0
    if a.cmd == "run" and (len(a.d) != 1 or len(a.eps) != 1):
        ap.error("run takes one --d and one --eps (use sweep)")
    for d in a.d:
        if not 2 <= d <= 12:
            ap.error("d must be in [2, 12]")
    rows = [run_case(a.case, d, eps, a.seed, a.save_u) for d in a.d for eps in a.eps]
    if a.out == "-":
        write_csv(sys.stdout, rows)
    else:
        tmp = a.out + ".tmp"
        write_csv(tmp, rows)
        os.replace(tmp, a.out)  # written atomically at the end
    return 0


if __name__ == "__main__":
    sys.exit(main())
