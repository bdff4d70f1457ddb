# Config-4 solve (2^10 x 2^10, variable E, upgraded AMEn): phase profile and ncu launch list.
set -x
mkdir -p gpurun_out
ARGS="--config 4 --trunc residual --rho 24 --local auto --rtol-factor 1e-3"
python tools/run_solve.py $ARGS > gpurun_out/solve_c4_plain.log 2>&1
QTT_SOLVER_PROFILE=1 python tools/run_solve.py $ARGS > gpurun_out/solve_c4_phases.log 2>&1
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/solve_c4_launches.csv \
    python tools/run_solve.py $ARGS > gpurun_out/solve_c4_ncu.log 2>&1
python tools/agg_launches.py gpurun_out/solve_c4_launches.csv > gpurun_out/solve_c4_launches.txt 2>&1
rm -f gpurun_out/solve_c4_launches.csv
tail -3 gpurun_out/solve_c4_plain.log | cut -c1-600
head -40 gpurun_out/solve_c4_launches.txt
