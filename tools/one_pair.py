"""Run matvec+round for one config-2 pair (used under ncu)."""
import sys
sys.path.insert(0, '.')
import torch
from bench import make_inputs, EPS
from paper_2501_07778_b200 import ttcore as T
rA, rx = (int(v) for v in sys.argv[1].split('x'))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
A, x = make_inputs(rA, rx)
TA, tx = T.TTMatrix(A), T.TTVector(x)
for _ in range(reps):
    z = T.tt_round(T.tt_matvec(TA, tx), EPS)
torch.cuda.synchronize()
print(z.ranks)
