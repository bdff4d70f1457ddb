mkdir -p gpurun_out
timeout 900 python tests/golden/make_conforming_gpu.py 10 > gpurun_out/g4_cg10.txt 2>&1
timeout 500 python tools/residual_floor.py 8 25 5 0.05 4 > gpurun_out/g4_f8_tf005.txt 2>&1
timeout 500 python tools/residual_floor.py 8 25 5 0.005 4 > gpurun_out/g4_f8_tf0005.txt 2>&1
cp gpurun_out/conforming_c5_d10.npz tests/golden/ 2>/dev/null
timeout 900 python tools/residual_floor.py 10 30 5 0.5 4 > gpurun_out/g4_f10.txt 2>&1
