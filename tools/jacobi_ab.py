"""A/B timing of the Jacobi SVD kernels through qtt_svd (square k x k inputs
with a spectrum that drops from 1 to 1e-13 over the first third and is
noise after that, like the assembly roundings).  Run once as is and once
with QTT_JACOBI_KERNEL=legacy."""
import ctypes, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2501_07778_b200 import _lib

for k in [int(a) for a in sys.argv[1:]] or (24, 60, 100, 150, 200, 224, 300, 400, 468, 600):
    rng = np.random.default_rng(k)
    u0, _ = np.linalg.qr(rng.standard_normal((k, k)))
    v0, _ = np.linalg.qr(rng.standard_normal((k, k)))
    s0 = np.concatenate([np.logspace(0, -13, k // 3), 1e-17 * rng.random(k - k // 3)])
    a = (u0 * s0) @ v0.T
    A = torch.tensor(a.ravel(order="F"), device="cuda")
    S = torch.zeros(k, dtype=torch.float64, device="cuda")
    U = torch.zeros(k * k, dtype=torch.float64, device="cuda")
    def run():
        _lib.call("qtt_svd", ctypes.c_int64(k), ctypes.c_int64(k), _lib.ptr(A), ctypes.c_int64(k),
                  _lib.ptr(S), _lib.ptr(U), ctypes.c_int64(k), _lib.stream_handle())
    run(); torch.cuda.synchronize()
    t = time.perf_counter(); n = 5
    for _ in range(n): run()
    torch.cuda.synchronize(); ms = (time.perf_counter() - t) / n * 1e3
    s = S.cpu().numpy(); sr = np.linalg.svd(a, compute_uv=False)
    uu = U.cpu().numpy().reshape(k, k).T
    top = k // 3
    orth = np.abs(uu[:, :top].T @ uu[:, :top] - np.eye(top)).max()
    print(f"k={k:4d} ms={ms:8.3f} max|ds|={np.abs(s - sr).max():.2e} orth(top)={orth:.1e}", flush=True)
