mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ttsvd.py tests/test_gpu_ttcore.py tests/test_gpu_scale.py tests/test_gpu_fem.py -q -k "decompose or ttsvd or config3 or low_rank or smooth or handoff or graded or mode_size or zero or golden or assembly or coupling" > gpurun_out/g10_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/g10_tests.txt
QTT_TTSVD_DEBUG=1 python tools/ttsvd_profile.py > gpurun_out/g10_debug.txt 2>&1
ncu --nvtx --nvtx-include "ttsvd/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g10_ttsvd_launches.csv python tools/ttsvd_profile.py > gpurun_out/g10_ncu.txt 2>&1
