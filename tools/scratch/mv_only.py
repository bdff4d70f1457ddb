import sys; sys.path.insert(0, '.')
import torch
from bench import make_inputs
from paper_2501_07778_b200 import ttcore as T
rA, rx = (int(v) for v in sys.argv[1].split('x'))
A, x = make_inputs(rA, rx)
TA, tx = T.TTMatrix(A), T.TTVector(x)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    y = T.tt_matvec(TA, tx)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); y = T.tt_matvec(TA, tx); e1.record(); torch.cuda.synchronize()
print("matvec ms", e0.elapsed_time(e1), "GB/s", 8 * sum(c.numel() for c in y.device_cores) / e0.elapsed_time(e1) / 1e6)
