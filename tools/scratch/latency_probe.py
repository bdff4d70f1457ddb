"""Back-to-back launch latency of small GEMMs (ours vs cuBLAS) with CUDA events."""
import ctypes, sys; sys.path.insert(0, ".")
import torch
from paper_2501_07778_b200 import _lib
S = _lib.stream_handle()
def t(fn, reps=200):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / reps * 1000
z = torch.zeros(1, device="cuda")
print("zero_ launch", round(t(lambda: z.zero_()), 2), "us")
for n in (64, 256, 1024, 1984):
    A = torch.randn(64, n, dtype=torch.float64, device="cuda"); C = torch.randn(n, n, dtype=torch.float64, device="cuda")
    ours = t(lambda: _lib.call("qtt_gemm", 1, 0, ctypes.c_int64(n), ctypes.c_int64(n), ctypes.c_int64(64), ctypes.c_double(-1.0), _lib.ptr(A), ctypes.c_int64(64), _lib.ptr(A), ctypes.c_int64(64), ctypes.c_double(1.0), _lib.ptr(C), ctypes.c_int64(n), S))
    cub = t(lambda: C.addmm_(A.T, A, alpha=-1.0))
    print("syrk n", n, "ours", round(ours, 2), "us  cublas", round(cub, 2), "us")
