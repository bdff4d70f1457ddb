"""GEMM shape histogram inside the config-4 AMEn solve (first sweeps; no
final compress so that the single-threaded GEMM profiler stays valid)."""
import sys, os, subprocess, collections
sys.path.insert(0, '.')
if os.environ.get('QTT_GEMM_LOG') is None:
    env = dict(os.environ, QTT_GEMM_LOG='1')
    r = subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, capture_output=True, text=True)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0]); tot = [0.0, 0.0]
    for line in r.stderr.splitlines():
        if not line.startswith('[gemm]'): continue
        m, n, k, b, fl, sp, t, f = line.split()[1:]
        key = (int(m) // 64 * 64, int(n) // 64 * 64, int(k) // 64 * 64, int(sp))
        a = agg[key]; a[0] += 1; a[1] += float(t); a[2] += float(f); tot[0] += float(t); tot[1] += float(f)
    print(r.stdout[-300:], r.stderr[-300:] if r.returncode else "")
    print(f"total GEMM {tot[0]:.1f} ms, {tot[1] / 1e9:.1f} GFLOP, {tot[1] / max(tot[0], 1e-9) / 1e9:.2f} TF/s")
    for key, (c, t, f) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
        print(f"{t:8.1f} ms {100 * t / tot[0]:5.1f}% x{c:6d} m~{key[0]:6d} n~{key[1]:6d} k~{key[2]:6d} sp={key[3]} {f / t / 1e9:6.2f} TF/s")
    sys.exit(0)
import torch
from paper_2501_07778_b200.configs import build_system
from paper_2501_07778_b200 import solver as S, _lib
gsys, eps = build_system(4, 10, {})
torch.cuda.synchronize()
_lib.gemm_profile_start()
S.solve(gsys.K, gsys.f, S.SolverConfig(epsilon=eps, seed=0, local_solver="auto", truncation="residual",
                                       enrichment_rank=24, local_rtol_factor=1e-3, max_sweeps=int(sys.argv[1]) if len(sys.argv) > 1 else 8))
torch.cuda.synchronize()
print(_lib.gemm_profile_stop())
