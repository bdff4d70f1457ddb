# AMEn enrichment-rank sweep on the config-4 variable-E 2^10 solve
export QTT_SOLVER_PROFILE=1
for rho in 16 24 32 48; do
  echo "=== rho $rho"
  QTT_AMEN_TRACE=1 timeout 900 python tools/run_solve.py --config 4 --d 10 --trunc residual --rho $rho --local auto --max-sweeps 40 2>&1 | grep -v "^\[amen\]" | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    if 'solve_s' in d: print({k: d[k] for k in ('solve_s', 'sweeps', 'residual', 'converged', 'rank_hist', 'profile')})
"
done
