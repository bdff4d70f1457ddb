"""Time qtt_qr on small shapes (run with and without QTT_NO_SMALLQR=1)."""
import ctypes, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2501_07778_b200 import _lib
for m, n in ((128, 64), (64, 64), (256, 32), (256, 64), (128, 16)):
    k = min(m, n)
    A = torch.randn(m * n, dtype=torch.float64, device="cuda")
    Q = torch.empty(m * k, dtype=torch.float64, device="cuda"); R = torch.empty(k * n, dtype=torch.float64, device="cuda")
    def run():
        _lib.call("qtt_qr", ctypes.c_int64(m), ctypes.c_int64(n), _lib.ptr(A), ctypes.c_int64(m), _lib.ptr(Q),
                  ctypes.c_int64(m), _lib.ptr(R), ctypes.c_int64(k), _lib.stream_handle())
    for _ in range(3): run()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(20): run()
    torch.cuda.synchronize(); print(f"{m}x{n}: {(time.perf_counter() - t) / 20 * 1e6:.1f} us", flush=True)
