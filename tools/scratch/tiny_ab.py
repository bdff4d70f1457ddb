"""A/B of the 32x32-tile GEMM threshold (QTT_GEMM_TINY_K) on the
latency-bound shapes of the rounding sweep: mean time per launch."""
import ctypes, os, sys, subprocess
sys.path.insert(0, '.')
SHAPES = [(512, 512, 512, 1, 4), (512, 512, 512, 1, 2), (256, 256, 256, 4, 4), (512, 512, 1024, 1, 0),
          (1024, 1024, 1024, 1, 4), (512, 512, 2048, 1, 1), (384, 384, 768, 1, 0)]
if len(sys.argv) == 1:
    for tk in ("512", "1100", "2100"):
        r = subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, QTT_GEMM_TINY_K=tk),
                           capture_output=True, text=True)
        print(f"TINY_K={tk}\n{r.stdout}{r.stderr[-800:]}")
    sys.exit(0)
import torch
from paper_2501_07778_b200 import _lib
_lib.load()
for m, n, k, batch, fl in SHAPES:
    A = torch.randn(m * k, dtype=torch.float64, device="cuda")
    B = torch.randn(k * n, dtype=torch.float64, device="cuda")
    C = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    def go():
        for _ in range(batch):
            _lib.call("qtt_gemm_structured", ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int64(m),
                      ctypes.c_int64(n), ctypes.c_int64(k), ctypes.c_double(1.0), _lib.ptr(A),
                      ctypes.c_int64(m), _lib.ptr(B), ctypes.c_int64(k), ctypes.c_double(0.0),
                      _lib.ptr(C), ctypes.c_int64(m), ctypes.c_int32(fl), _lib.stream_handle())
    for _ in range(5): go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): go()
    e1.record(); torch.cuda.synchronize()
    print(f"m={m} n={n} k={k} x{batch} fl={fl}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us")
