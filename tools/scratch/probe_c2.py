import sys, time, json
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2501_07778_b200 import ttcore as T

def make(rA, rx, d=24):
    rngA = np.random.default_rng(1000 + rA)
    ra = [1] + [rA] * (d - 1) + [1]
    A = [rngA.standard_normal((ra[k], 2, 2, ra[k + 1])) / np.sqrt(rA) for k in range(d)]
    rngx = np.random.default_rng(2000 + rx)
    rc = [1] + [rx] * (d - 1) + [1]
    x = [rngx.standard_normal((rc[k], 2, rc[k + 1])) / np.sqrt(rx) for k in range(d)]
    return A, x

pairs = [(a, b) for a in (4, 8, 16) for b in (16, 64, 128)]
if len(sys.argv) > 1:
    pairs = [tuple(int(v) for v in p.split('x')) for p in sys.argv[1:]]
for rA, rx in pairs:
    A, x = make(rA, rx)
    TA, tx = T.TTMatrix(A), T.TTVector(x)
    torch.cuda.synchronize()
    for it in range(2):
        t0 = time.perf_counter(); y = T.tt_matvec(TA, tx); torch.cuda.synchronize(); t1 = time.perf_counter()
        z = T.tt_round(y, 1e-10); torch.cuda.synchronize(); t2 = time.perf_counter()
    R = rA * rx
    caps = tuple([1] + [min(R, 2**k, 2**(24 - k)) for k in range(1, 24)] + [1])
    print(json.dumps({"pair": f"{rA}x{rx}", "matvec_ms": (t1 - t0) * 1e3, "round_ms": (t2 - t1) * 1e3,
                      "ranks_ok": z.ranks == caps, "maxrank": max(z.ranks)}), flush=True)
