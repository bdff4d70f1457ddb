"""Launch list of one config-3 TT-SVD (2^26 field, eps=1e-8), nvtx range 'ttsvd'."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2501_07778_b200 import ttcore as T
from paper_2501_07778_b200.assembly import _flat_ordered
n = 1 << 13
xs = torch.arange(n, dtype=torch.float64, device='cuda') / (n - 1)
X, Y = torch.meshgrid(xs, xs, indexing='ij')
v = _flat_ordered(torch.sin(3 * X) * torch.exp(-Y) + 0.1 * torch.cos(7 * X * Y), 'zorder')
T.tt_decompose(v, 1e-8)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("ttsvd")
t = T.tt_decompose(v, 1e-8)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print(t.ranks)
