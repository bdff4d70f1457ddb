# Round-end measurement artefacts (run on the GPU box from the repo root):
# bench line, ncu launch list of the config-2 step, full captures of the
# top DMMA GEMM launch and of the matvec kernel.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/step_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/ncu_step.log 2>&1
python tools/agg_launches.py gpurun_out/step_launches.csv > gpurun_out/step_launches.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 400 -c 1 \
    -o gpurun_out/gemm_full python tools/one_pair.py 16x128 1 > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none -k regex:core_product_kernel -c 1 \
    -o gpurun_out/mv_full python tools/one_pair.py 16x128 1 > gpurun_out/ncu_mv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi_ring -s 30 -c 1 \
    -o gpurun_out/jring_full python tools/jacobi_ab.py 200 > gpurun_out/ncu_jr.log 2>&1
ls -la gpurun_out
