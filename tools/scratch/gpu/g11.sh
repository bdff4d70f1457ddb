mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ttsvd.py tests/test_gpu_scale.py -q -k "ttsvd or config3 or low_rank or smooth or handoff or graded or mode_size or zero" > gpurun_out/g11_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/g11_tests.txt
ncu --nvtx --nvtx-include "ttsvd/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g11_ttsvd_launches.csv python tools/ttsvd_profile.py > gpurun_out/g11_ncu.txt 2>&1
ncu --nvtx --nvtx-include "ttsvd/" -c 3 --set full --import-source on --clock-control none -o gpurun_out/g11_full -f python tools/ttsvd_profile.py > gpurun_out/g11_ncu2.txt 2>&1
