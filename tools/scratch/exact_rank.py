"""Analysis: QTT ranks of the exact (dense-solved) solution of a config at
small d, to see whether AMEn rank growth is intrinsic."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2501_07778_b200.configs import build_system
from paper_2501_07778_b200 import ttcore as T
idx, d = int(sys.argv[1]), int(sys.argv[2])
T._CONTRACT_GUARD_BITS = 30
gsys, eps = build_system(idx, d)
K = T.tt_contract_device(gsys.K); f = T.tt_contract_device(gsys.f)
u = torch.linalg.solve(K, f)
for tol in (1e-6, 1e-8, 1e-10):
    print(idx, d, tol, T.tt_decompose(u, tol).ranks)
