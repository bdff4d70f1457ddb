"""Per-iteration cost of the native local GMRES / local apply at AMEn-like
shapes (rl = rr = r, n = 2, K rank 117)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2501_07778_b200 import solver as S

for r in [int(a) for a in (sys.argv[1:] or ["66", "130", "260"])]:
    ra = rb = 117; n = 2
    rng = np.random.default_rng(r)
    pl = torch.tensor(rng.standard_normal((r, ra, r)) / r, device="cuda")
    pr = torch.tensor(rng.standard_normal((r, rb, r)) / r, device="cuda")
    a = rng.standard_normal((ra, n, n, rb))
    ap = {"ra": ra, "rb": rb, "aj_ib": torch.tensor(a.transpose(0, 2, 1, 3).reshape(ra * n, n * rb).copy(), device="cuda")}
    x = torch.tensor(rng.standard_normal((r, n, r)), device="cuda")
    for _ in range(3): S._local_matvec(pl, ap, pr, x)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(20): S._local_matvec(pl, ap, pr, x)
    torch.cuda.synchronize(); tmv = (time.perf_counter() - t) / 20
    S._gmres(pl, ap, pr, x, torch.zeros_like(x), 0.0, maxit=40)
    torch.cuda.synchronize(); t = time.perf_counter()
    _, ok, its = S._gmres(pl, ap, pr, x, torch.zeros_like(x), 0.0, maxit=80)
    torch.cuda.synchronize(); tg = (time.perf_counter() - t) / max(its, 1)
    fl = 2 * r * ra * r * n * r * 2 + 2 * r * r * ra * n * n * rb
    print(f"r={r} dim={r*n*r} matvec {tmv*1e3:.3f} ms ({fl/tmv/1e12:.1f} TF/s)  gmres/it {tg*1e3:.3f} ms its={its}", flush=True)
