"""GEMM shape histogram of one config-2 pair's tt_round (QTT_GEMM_LOG=1):
time and executed flops per (m, n, k, flags) class."""
import sys, os, subprocess, collections
sys.path.insert(0, '.')
if os.environ.get('QTT_GEMM_LOG') is None:
    env = dict(os.environ, QTT_GEMM_LOG='1')
    r = subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, capture_output=True, text=True)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0]); tot = [0.0, 0.0]
    for line in r.stderr.splitlines():
        if not line.startswith('[gemm]'): continue
        m, n, k, b, fl, sp, t, f = line.split()[1:]
        key = (int(m), int(n), int(k), int(fl), int(sp))
        a = agg[key]; a[0] += 1; a[1] += float(t); a[2] += float(f); tot[0] += float(t); tot[1] += float(f)
    print(r.stdout[-500:])
    print(f"total GEMM {tot[0]:.2f} ms, {tot[1] / 1e9:.1f} GFLOP, {tot[1] / tot[0] / 1e9:.2f} TF/s")
    for key, (c, t, f) in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
        print(f"{t:8.3f} ms {100 * t / tot[0]:5.1f}% x{c:5d} m={key[0]:6d} n={key[1]:6d} k={key[2]:6d} fl={key[3]} sp={key[4]} {f / t / 1e9:6.2f} TF/s")
    sys.exit(r.returncode)
import torch
from bench import make_inputs, EPS
from paper_2501_07778_b200 import ttcore as T, _lib
rA, rx = (int(v) for v in sys.argv[1].split('x'))
A, x = make_inputs(rA, rx); TA, tx = T.TTMatrix(A), T.TTVector(x)
for _ in range(2): z = T.tt_round(T.tt_matvec(TA, tx), EPS)
torch.cuda.synchronize()
y = T.tt_matvec(TA, tx); torch.cuda.synchronize()
_lib.gemm_profile_start(); z = T.tt_round(y, EPS); print(_lib.gemm_profile_stop())
