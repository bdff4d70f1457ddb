mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 100 -c 1 \
    -o gpurun_out/gemm_full python tools/one_pair.py 16x128 1 > gpurun_out/ncu_gemm.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:core_product_kernel -c 1 \
    -o gpurun_out/mv_full python tools/one_pair.py 16x128 1 > gpurun_out/ncu_mv.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:jacobi_ring -s 30 -c 1 \
    -o gpurun_out/jring_full python tools/jacobi_ab.py 200 > gpurun_out/ncu_jr.log 2>&1
ls -la gpurun_out
