# Round-end measurement artefacts (run on the GPU box from the repo root):
# bench line, ncu launch list of one config-2 step, ncu --set full captures of the
# top DMMA GEMM launch, the matvec kernel and the fused small factor kernel.
set -x
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/step_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/ncu_step.log 2>&1
python tools/agg_launches.py gpurun_out/step_launches.csv > gpurun_out/step_launches.txt 2>&1
rm -f gpurun_out/step_launches.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 60 -c 40 \
    -o gpurun_out/gemm_full python tools/one_pair.py 16x128 1 > gpurun_out/ncu_gemm.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:core_product_kernel -c 1 \
    -o gpurun_out/mv_full python tools/one_pair.py 16x128 1 > gpurun_out/ncu_mv.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:chol_inv_small2 -s 10 -c 2 \
    -o gpurun_out/cis_full python tools/c3_round.py 1 > gpurun_out/ncu_cis.log 2>&1
for rep in gemm_full mv_full cis_full; do
  ncu -i gpurun_out/$rep.ncu-rep --page raw --csv > gpurun_out/$rep.csv 2>/dev/null
done
python tools/ncu_summary.py gpurun_out/gemm_full.csv gpurun_out/mv_full.csv gpurun_out/cis_full.csv > gpurun_out/kernel_evidence.txt 2>&1
ls -la gpurun_out
