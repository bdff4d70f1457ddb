"""Config-3 rounding input (d=26, sum of 16 rank-8 terms) rounded REPS times (timing / ncu / trace)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2501_07778_b200 import ttcore as T
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rng = np.random.default_rng(3000)
acc = None
for _ in range(16):
    rk = [1] + [8] * 25 + [1]
    t = T.TTVector([rng.standard_normal((rk[k], 2, rk[k + 1])) / np.sqrt(8) for k in range(26)])
    acc = t if acc is None else T.tt_add(acc, t)
for _ in range(reps):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); z = T.tt_round(acc, 1e-10); e1.record(); torch.cuda.synchronize()
    print("round ms", round(e0.elapsed_time(e1), 3), flush=True)
print(max(z.ranks))
