mkdir -p gpurun_out
timeout 600 python tools/residual_floor.py 6 30 > gpurun_out/g3_floor6.txt 2>&1
timeout 600 python tools/residual_floor.py 8 12 > gpurun_out/g3_floor8.txt 2>&1
timeout 600 python tools/residual_floor.py 7 12 > gpurun_out/g3_floor7.txt 2>&1
python tools/ttsvd_profile.py > gpurun_out/g3_plain.txt 2>&1
ncu --nvtx --nvtx-include "ttsvd/" --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/g3_ttsvd_launches.csv python tools/ttsvd_profile.py > gpurun_out/g3_ncu.txt 2>&1
python tools/agg_launches.py gpurun_out/g3_ttsvd_launches.csv > gpurun_out/g3_agg.txt 2>&1
