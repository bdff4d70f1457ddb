mkdir -p gpurun_out
QTT_TTSVD_DEBUG=1 python tools/ttsvd_profile.py > gpurun_out/g8_debug.txt 2>&1
ncu --nvtx --nvtx-include "ttsvd/" -c 2 --set full --import-source on --clock-control none -o gpurun_out/g8_ttsvd_full -f python tools/ttsvd_profile.py > gpurun_out/g8_ncu.txt 2>&1
