"""qtt_dense_solve timing vs N (SPD-like diagonally dominant matrices)."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2501_07778_b200._dense import dense_solve_colmajor
for n in [int(a) for a in sys.argv[1:]] or (1024, 2048, 3200, 4096, 6050, 8192):
    g = torch.Generator(device="cuda").manual_seed(n)
    m = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g) / n ** 0.5
    m = m @ m.T + torch.eye(n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    mc = m.contiguous().view(-1)
    for _ in range(2): x, fb = dense_solve_colmajor(mc, n, b)
    torch.cuda.synchronize(); t = time.perf_counter(); reps = 5
    for _ in range(reps): x, fb = dense_solve_colmajor(mc, n, b)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / reps
    res = float(torch.linalg.vector_norm(m @ x - b) / torch.linalg.vector_norm(b))
    print(f"N={n} {dt*1e3:.2f} ms  {(2/3)*n**3/dt/1e12:.1f} TF/s  res {res:.1e} fb {fb}", flush=True)
