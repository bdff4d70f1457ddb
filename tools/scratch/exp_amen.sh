export QTT_SOLVER_PROFILE=1
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
echo "=== asm profile d10"; timeout 300 python tools/asm_profile.py 10 2>&1 | tail -12
echo "=== config5 d10 auto rho16"; QTT_AMEN_TRACE=1 timeout 1200 python tools/run_solve.py --config 5 --d 10 --trunc residual --rho 16 --local auto --max-sweeps 40 --dense-bits 23 2>&1 | cut -c1-2500
