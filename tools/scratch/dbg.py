import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_2501_07778_b200._dense import dense_solve_colmajor
rng = np.random.default_rng(11)
for n in [int(v) for v in sys.argv[1:]]:
    a = rng.standard_normal((n, n)); m = a @ a.T + n * np.eye(n); b = rng.standard_normal(n)
    x, fb = dense_solve_colmajor(torch.tensor(m.T.ravel(), device="cuda"), n, torch.tensor(b, device="cuda"))
    print(n, fb, np.linalg.norm(m @ x.cpu().numpy() - b))
m = np.array([[0.0, 1.0], [1.0, 0.0]])
x, fb = dense_solve_colmajor(torch.tensor(m.T.ravel(), device="cuda"), 2, torch.tensor([1.0, 2.0], device="cuda"))
print(fb, x.cpu().numpy())
