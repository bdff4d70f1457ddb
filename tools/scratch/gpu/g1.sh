mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/g1_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/g1_tests.txt
QTT_AMEN_TRACE=1 timeout 600 python tools/run_solve.py --config 5 --d 8 --trunc residual --rho 24 --local auto --rtol-factor 1e-3 --max-sweeps 30 > gpurun_out/g1_c5d8.txt 2>&1
