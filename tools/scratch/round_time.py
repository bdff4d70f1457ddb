import sys; sys.path.insert(0, ".")
import torch
from bench import make_inputs, EPS
from paper_2501_07778_b200 import ttcore as T
pairs = [tuple(int(v) for v in p.split("x")) for p in sys.argv[1:]] or [(16,128),(8,128),(16,64),(4,128)]
for p in pairs:
    A, x = make_inputs(*p); TA, tx = T.TTMatrix(A), T.TTVector(x)
    y = T.tt_matvec(TA, tx); z = T.tt_round(y, EPS); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); z = T.tt_round(y, EPS); e1.record(); torch.cuda.synchronize()
    print(p, "round ms", round(e0.elapsed_time(e1), 2), flush=True)
