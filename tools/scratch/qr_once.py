import ctypes, sys; sys.path.insert(0, ".")
import torch
from paper_2501_07778_b200 import _lib
m, n = int(sys.argv[1]), int(sys.argv[2])
A = torch.randn(m * n, dtype=torch.float64, device="cuda"); Q = torch.empty(m * n, dtype=torch.float64, device="cuda"); R = torch.empty(n * n, dtype=torch.float64, device="cuda")
for _ in range(2):
    _lib.call("qtt_qr", ctypes.c_int64(m), ctypes.c_int64(n), _lib.ptr(A), ctypes.c_int64(m), _lib.ptr(Q), ctypes.c_int64(m), _lib.ptr(R), ctypes.c_int64(n), _lib.stream_handle())
torch.cuda.synchronize(); print("ok")
