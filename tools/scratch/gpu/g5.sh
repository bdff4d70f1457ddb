mkdir -p gpurun_out
timeout 600 python tools/residual_floor.py 8 25 5 0.5 4 0 > gpurun_out/g5_f8_r0.txt 2>&1
timeout 600 python tools/residual_floor.py 8 25 5 0.05 4 0 > gpurun_out/g5_f8_r0_tf005.txt 2>&1
timeout 900 python tools/residual_floor.py 10 30 5 0.5 4 0 > gpurun_out/g5_f10_r0.txt 2>&1
timeout 900 python tools/residual_floor.py 10 30 5 0.05 4 0 > gpurun_out/g5_f10_r0_tf005.txt 2>&1
