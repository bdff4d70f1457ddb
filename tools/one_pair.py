"""Run matvec+round for one config-2 pair (used under ncu); with TRACE=1 the
last repetition prints the per-phase timings of the rounding (QTT_ROUND_TRACE)."""
import os
import sys
sys.path.insert(0, '.')
import torch
from bench import make_inputs, EPS
from paper_2501_07778_b200 import ttcore as T
rA, rx = (int(v) for v in sys.argv[1].split('x'))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
A, x = make_inputs(rA, rx)
TA, tx = T.TTMatrix(A), T.TTVector(x)
for i in range(reps):
    if i == reps - 1 and os.environ.get("TRACE"):
        os.environ["QTT_ROUND_TRACE"] = "1"
        os.environ["QTT_CERT_DEBUG"] = "1"
    y = T.tt_matvec(TA, tx)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); z = T.tt_round(y, EPS); e1.record(); torch.cuda.synchronize()
    print("round ms", round(e0.elapsed_time(e1), 3), flush=True)
print(z.ranks)
