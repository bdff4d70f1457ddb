"""One DMMA GEMM of a given shape through the C ABI (for ncu): m n k."""
import sys; sys.path.insert(0, ".")
import torch
from paper_2501_07778_b200._dense import mm
m, n, k = (int(v) for v in sys.argv[1:4])
a = torch.randn(m, k, dtype=torch.float64, device="cuda"); b = torch.randn(k, n, dtype=torch.float64, device="cuda")
for _ in range(2): c = mm(a, b)
torch.cuda.synchronize(); print("ok")
