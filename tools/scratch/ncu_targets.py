"""Small driver for single-kernel ncu captures: a large DMMA GEMM and the
config-2 16x128 matvec."""
import sys; sys.path.insert(0, ".")
import torch
from paper_2501_07778_b200._dense import mm
from bench import make_inputs
from paper_2501_07778_b200 import ttcore as T
which = sys.argv[1]
if which == "gemm":
    a = torch.randn(4096, 2048, dtype=torch.float64, device="cuda"); b = torch.randn(2048, 2048, dtype=torch.float64, device="cuda")
    for _ in range(3): mm(a, b)
else:
    A, x = make_inputs(16, 128); TA, tx = T.TTMatrix(A), T.TTVector(x)
    for _ in range(3): T.tt_matvec(TA, tx)
torch.cuda.synchronize(); print("ok")
