"""BASELINE config 3: rounding of a 16-term rank-8 sum (d=26, R=128) and the
TT-SVD of g(x,y) on a 2^13 x 2^13 Z-ordered grid (2^26 entries)."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2501_07778_b200 import ttcore as T

def rounding_input(d=26, terms=16, r=8, seed=3000):
    rng = np.random.default_rng(seed)
    acc = None
    for _ in range(terms):
        rk = [1] + [r] * (d - 1) + [1]
        t = T.TTVector([rng.standard_normal((rk[k], 2, rk[k + 1])) / np.sqrt(r) for k in range(d)])
        acc = t if acc is None else T.tt_add(acc, t)
    return acc

def field(bits=13):
    n = 1 << bits
    xs = torch.arange(n, dtype=torch.float64, device='cuda') / (n - 1)
    X, Y = torch.meshgrid(xs, xs, indexing='ij')
    g = torch.sin(3 * X) * torch.exp(-Y) + 0.1 * torch.cos(7 * X * Y)
    from paper_2501_07778_b200.assembly import _flat_ordered
    return _flat_ordered(g, 'zorder')

out = {}
t = rounding_input()
torch.cuda.synchronize()
for eps in (1e-6, 1e-10):
    for rep in range(2):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); r = T.tt_round(t, eps); e1.record(); torch.cuda.synchronize()
    out[f'round_{eps}'] = {'ms': e0.elapsed_time(e1), 'ranks_max': max(r.ranks), 'ranks': r.ranks}
v = field()
for rep in range(2):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); tv = T.tt_decompose(v, 1e-8); e1.record(); torch.cuda.synchronize()
out['ttsvd'] = {'ms': e0.elapsed_time(e1), 'ranks': tv.ranks}
# accuracy of the TT-SVD on a sample of entries (full contraction would be 2^26)
print(json.dumps(out))
