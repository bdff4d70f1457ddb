# Per-kernel ncu evidence (duration, DRAM bytes, FP64 pipe, DMMA instructions)
# over representative workloads; summarised by tools/kernel_evidence.py.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
run() { timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ev_$1.csv "${@:2}" > /dev/null 2>&1; echo "$1 rc=$?"; }
run pair python tools/one_pair.py 16x128 1
run jac python tools/jacobi_ab.py 200 468
run qr python tools/qr_small_bench.py
run gmres python tools/gmres_micro.py 130
run lu python tools/lu_bench.py 4096
python tools/kernel_evidence.py gpurun_out/ev_*.csv > gpurun_out/kernel_evidence.txt
cat gpurun_out/kernel_evidence.txt
