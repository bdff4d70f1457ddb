export QTT_AMEN_TRACE=1 QTT_SOLVER_PROFILE=1
mkdir -p gpurun_out
echo "=== d8 auto rho16"; timeout 600 python tools/run_solve.py --config 4 --d 8 --trunc residual --rho 16 --local auto 2>&1 | cut -c1-2500
echo "=== d10 auto rho16"; timeout 1500 python tools/run_solve.py --config 4 --d 10 --trunc residual --rho 16 --local auto --max-sweeps 40 2>&1 | cut -c1-2500
