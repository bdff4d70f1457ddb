import sys; sys.path.insert(0, ".")
import torch
from paper_2501_07778_b200._dense import mm
for (m, n, k) in [(4096, 4096, 4096), (4096, 2048, 2048), (4096, 2048, 32), (32, 2048, 4096), (8192, 8192, 8192), (6000, 6000, 64)]:
    a = torch.randn(m, k, dtype=torch.float64, device="cuda"); b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    c = mm(a, b); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): c = mm(a, b)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 5
    e0.record()
    for _ in range(5): c2 = a @ b
    e1.record(); torch.cuda.synchronize()
    t2 = e0.elapsed_time(e1) / 5
    print((m, n, k), "ours TF/s", round(2 * m * n * k / t / 1e9, 2), "cublas TF/s", round(2 * m * n * k / t2 / 1e9, 2), "maxdiff", float((c - c2).abs().max()))
