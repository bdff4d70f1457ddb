"""A/B micro-benchmark: dense_solve and qr through two builds of the library."""
import ctypes, sys; sys.path.insert(0, ".")
import numpy as np, torch
libs = {"new": ctypes.CDLL("paper_2501_07778_b200/lib/libqttb200.so"), "old": ctypes.CDLL("tools/old_libqttb200.so")}
S = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / reps
rng = np.random.default_rng(0)
for n in (2000, 6000):
    a = rng.standard_normal((n, n)); m = a @ a.T / n + np.eye(n)
    M = torch.tensor(m.T.ravel(), device="cuda"); b = torch.tensor(rng.standard_normal(n), device="cuda"); x = torch.empty(n, dtype=torch.float64, device="cuda"); fb = ctypes.c_int32()
    for k, L in libs.items():
        ms = t(lambda: L.qtt_dense_solve(ctypes.c_int64(n), ctypes.c_void_p(M.data_ptr()), ctypes.c_int64(n), ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(x.data_ptr()), ctypes.byref(fb), S))
        print("dense_solve", n, k, round(ms, 2), "ms", flush=True)
for (mm, nn) in ((4096, 2048), (2048, 2048)):
    A = torch.randn(mm * nn, dtype=torch.float64, device="cuda"); Q = torch.empty(mm * nn, dtype=torch.float64, device="cuda"); R = torch.empty(nn * nn, dtype=torch.float64, device="cuda")
    for k, L in libs.items():
        ms = t(lambda: L.qtt_qr(ctypes.c_int64(mm), ctypes.c_int64(nn), ctypes.c_void_p(A.data_ptr()), ctypes.c_int64(mm), ctypes.c_void_p(Q.data_ptr()), ctypes.c_int64(mm), ctypes.c_void_p(R.data_ptr()), ctypes.c_int64(nn), S))
        print("qr", mm, nn, k, round(ms, 2), "ms", flush=True)
