"""Measure FP64 peaks on the B200 box (DGEMM via cuBLAS as the DMMA roof)."""
import json, os, time
import torch

def main():
    out = {"cpu_count": os.cpu_count()}
    try:
        import threadpoolctl
        out["blas"] = [{k: v for k, v in d.items() if k in ("internal_api", "num_threads", "version")}
                       for d in threadpoolctl.threadpool_info()]
    except Exception as e:  # pragma: no cover
        out["blas"] = str(e)
    dev = torch.device("cuda:0")
    out["gpu"] = torch.cuda.get_device_name(0)
    out["sms"] = torch.cuda.get_device_properties(0).multi_processor_count
    for n in (2048, 4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device=dev)
        b = torch.randn(n, n, dtype=torch.float64, device=dev)
        for _ in range(3):
            c = a @ b
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            s.record(); c = a @ b; e.record(); torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e) / 1e3)
        out[f"dgemm_{n}_tflops"] = 2 * n**3 / best / 1e12
    x = torch.empty(1 << 28, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    for _ in range(3):
        y.copy_(x)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); y.copy_(x); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    out["copy_gbs"] = 2 * x.numel() * 8 / best / 1e9
    import numpy as np
    a = np.random.default_rng(0).standard_normal((2048, 2048))
    t = time.perf_counter(); np.linalg.qr(a); out["cpu_qr2048_s"] = time.perf_counter() - t
    t = time.perf_counter(); a @ a; out["cpu_gemm2048_s"] = time.perf_counter() - t
    print(json.dumps(out))

if __name__ == "__main__":
    main()
