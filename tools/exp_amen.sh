export QTT_AMEN_TRACE=1 QTT_SOLVER_PROFILE=1
mkdir -p gpurun_out
echo "=== d8 rho8 random"; timeout 600 python tools/run_solve.py --config 4 --d 8 --trunc residual --rho 8 2>&1 | grep -v "^\[amen\]" | cut -c1-3000
echo "=== d8 rho16 random"; timeout 600 python tools/run_solve.py --config 4 --d 8 --trunc residual --rho 16 2>&1 | tail -1 | cut -c1-3000
echo "=== nested 6->8 rho8"; timeout 900 python tools/nested.py --d0 6 --d1 8 --rho 8 2>&1 | grep -v "^\[amen\]"
echo "=== nested 6->8 rho8 init 1e-7"; timeout 900 python tools/nested.py --d0 6 --d1 8 --rho 8 --init-eps 1e-7 2>&1 | grep -v "^\[amen\]"
echo "=== gemm shapes 16x128"; timeout 300 python tools/gemm_shapes.py 16x128 2>&1 | tail -45
