mkdir -p gpurun_out
make -j16 > gpurun_out/g6_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ttsvd.py tests/test_gpu_ttcore.py tests/test_gpu_fem.py tests/test_gpu_scale.py -q -x -k "decompose or ttsvd or config3 or golden or assembly or coupling or low_rank or smooth or handoff or graded or mode_size or zero" > gpurun_out/g6_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/g6_tests.txt
python tools/ttsvd_profile.py > gpurun_out/g6_plain.txt 2>&1
python - > gpurun_out/g6_time.txt 2>&1 <<'PY'
import sys; sys.path.insert(0,'.')
import torch
from paper_2501_07778_b200 import ttcore as T
from paper_2501_07778_b200.assembly import _flat_ordered
n = 1 << 13
xs = torch.arange(n, dtype=torch.float64, device='cuda') / (n - 1)
X, Y = torch.meshgrid(xs, xs, indexing='ij')
v = _flat_ordered(torch.sin(3 * X) * torch.exp(-Y) + 0.1 * torch.cos(7 * X * Y), 'zorder')
for _ in range(2): T.tt_decompose(v, 1e-8)
torch.cuda.synchronize()
for _ in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); t = T.tt_decompose(v, 1e-8); e1.record(); torch.cuda.synchronize()
    print('ttsvd ms', e0.elapsed_time(e1), t.ranks)
PY
ncu --nvtx --nvtx-include "ttsvd/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g6_ttsvd_launches.csv python tools/ttsvd_profile.py > gpurun_out/g6_ncu.txt 2>&1
python tools/agg_launches.py gpurun_out/g6_ttsvd_launches.csv > gpurun_out/g6_agg.txt 2>&1
timeout 900 python tools/qtt_cg_exact.py 5 8 > gpurun_out/g6_cg8.txt 2>&1
