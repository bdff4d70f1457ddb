mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/g2_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/g2_tests.txt
run() { name=$1; shift; QTT_AMEN_TRACE=1 timeout 300 python tools/run_solve.py "$@" > gpurun_out/g2_$name.txt 2>&1; }
run d6ref --config 5 --d 6 --trunc reference --rho 4 --local direct --max-sweeps 40
run d7res --config 5 --d 7 --trunc residual --rho 24 --local auto --rtol-factor 1e-3 --max-sweeps 30
run d8rho64 --config 5 --d 8 --trunc residual --rho 64 --local auto --rtol-factor 1e-3 --max-sweeps 25
run d8strict --config 5 --d 8 --trunc residual --rho 24 --local auto --rtol-factor 0 --max-sweeps 25
run d8tf01 --config 5 --d 8 --trunc residual --rho 24 --local auto --rtol-factor 1e-3 --trunc-factor 0.1 --max-sweeps 25
run d8direct --config 5 --d 8 --trunc residual --rho 24 --local direct --max-sweeps 20
