"""Prototype (diagnostics only, torch on the device): GMRES iteration counts
for AMEn local systems of the variable-E config-4 solve under candidate
preconditioners.  Captures local systems through solver._LOCAL_HOOK."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2501_07778_b200.configs import build_system
from paper_2501_07778_b200 import solver as S
d = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cap = []
def hook(phi_l, a_p, phi_r, rhs, x_cur, sol):
    if rhs.numel() > 15000 and x_cur is not None and x_cur.shape == rhs.shape:
        cap.append([t.clone() for t in (phi_l, a_p["a_ijb"].view(a_p["ra"], a_p["n"], a_p["n"], a_p["rb"]), phi_r, rhs, x_cur, sol)])
        if len(cap) > 6: cap.pop(0)
gsys, eps = build_system(4, d)
S._LOCAL_HOOK = None
out = S.solve(gsys.K, gsys.f, S.SolverConfig(epsilon=eps, seed=0, truncation='residual', enrichment_rank=16, max_sweeps=5))
print('pre-solve', out.residual_history, flush=True)
S._LOCAL_HOOK = hook
out = S.solve(gsys.K, gsys.f, S.SolverConfig(epsilon=eps, seed=0, truncation='residual', enrichment_rank=16, max_sweeps=7))
print('captured', len(cap), out.residual_history[-2:], flush=True)

def mv_factory(Pl, A, Pr):
    def mv(x):
        t1 = torch.einsum('xay,yjh->xajh', Pl, x)
        t2 = torch.einsum('xajh,aijb->xibh', t1, A)
        return torch.einsum('xibh,gbh->xig', t2, Pr)
    return mv

def gmres(mv, prec, b, x0, tol, m=40, maxit=600):
    x = x0.clone(); bn = float(torch.linalg.vector_norm(b)); hist = []
    it = 0
    while it < maxit:
        r = b - mv(x); rn = float(torch.linalg.vector_norm(r)); hist.append(rn / bn)
        if rn / bn <= tol: break
        V = [r / rn]; Z = []; H = torch.zeros(m + 1, m, dtype=torch.float64, device=b.device)
        g = torch.zeros(m + 1, dtype=torch.float64, device=b.device); g[0] = rn
        for j in range(m):
            z = prec(V[j]); Z.append(z); w = mv(z)
            for _ in range(2):
                for i in range(j + 1):
                    h = torch.sum(w * V[i]); H[i, j] += h; w = w - h * V[i]
            H[j + 1, j] = torch.linalg.vector_norm(w); V.append(w / H[j + 1, j]); it += 1
            y = torch.linalg.lstsq(H[:j + 2, :j + 1], g[:j + 2, None]).solution[:, 0]
            res = float(torch.linalg.vector_norm(g[:j + 2] - H[:j + 2, :j + 1] @ y))
            if res / bn <= tol or it >= maxit: break
        for i in range(len(Z)): x = x + y[i] * Z[i]
    return x, it, hist

def kron2(Pl, A, Pr, split):
    ra = A.shape[0]; rb = A.shape[3]
    # M = sum_b L_b (x) R_b (split 'xi|g') with L_b = sum_a Pl_a (x) A_ab
    GPl = torch.einsum('xay,xcy->ac', Pl, Pl)
    if split == 'xi|g':
        GA = torch.einsum('aijb,cijd->acbd', A, A)
        GL = torch.einsum('ac,acbd->bd', GPl, GA)
        GR = torch.einsum('gbh,gdh->bd', Pr, Pr)
    def isqrt(G):
        w, V = torch.linalg.eigh(G); keep = w > w.max() * 1e-14
        return V[:, keep] * w[keep].sqrt(), V[:, keep] / w[keep].sqrt()
    FL, FLi = isqrt(GL); FR, FRi = isqrt(GR)
    U, s, Vh = torch.linalg.svd(FL.T @ FR)
    alpha = [FLi @ U[:, t] * s[t] for t in range(2)]
    beta = [FRi @ Vh[t] for t in range(2)]
    L = [torch.einsum('xay,aijb,b->xiyj', Pl, A, al).reshape(Pl.shape[0] * A.shape[1], -1) for al in alpha]
    R = [torch.einsum('gbh,b->gh', Pr, be) for be in beta]
    # P vec(Z) = L1 Z R1^T + L2 Z R2^T  (Z: (x i) x g)
    T = torch.linalg.solve(R[0].T, R[1].T)  # R1^{-T} R2^T
    lam, W = torch.linalg.eig(T)
    Wi = torch.linalg.inv(W)
    Lc = [l.to(torch.complex128) for l in L]
    blocks = torch.stack([Lc[0] + lam[j] * Lc[1] for j in range(lam.shape[0])])
    LU, piv = torch.linalg.lu_factor(blocks)
    R1iT = torch.linalg.inv(R[0]).T
    nxi = L[0].shape[0]
    def prec(v):
        V = v.reshape(nxi, -1).to(torch.complex128)
        rhs = V @ W  # columns j
        Y = torch.linalg.lu_solve(LU, piv, rhs.T.unsqueeze(2))[:, :, 0].T  # (nxi, g)
        Yr = (Y @ Wi).real
        return (Yr @ R1iT).reshape(v.shape)
    rel = float(s[2] / s[0]) if s.numel() > 2 else 0.0
    return prec, rel

def dense32(Pl, A, Pr):
    M = torch.einsum('xay,aijb,gbh->xigyjh', Pl, A, Pr)
    n = Pl.shape[0] * A.shape[1] * Pr.shape[0]
    M = M.reshape(n, n).float(); LU, piv = torch.linalg.lu_factor(M); del M
    def prec(v):
        return torch.linalg.lu_solve(LU, piv, v.reshape(-1, 1).float()).double().reshape(v.shape)
    return prec

for ci, (Pl, A, Pr, rhs, xc, sol) in enumerate(cap[-3:]):
    mv = mv_factory(Pl, A, Pr)
    bn = float(torch.linalg.vector_norm(rhs))
    chk = float(torch.linalg.vector_norm(mv(sol) - rhs)) / bn
    r0 = float(torch.linalg.vector_norm(mv(xc) - rhs)) / bn
    info = {'shape': tuple(rhs.shape), 'rA': (A.shape[0], A.shape[3]), 'sol_res': chk, 'warm_res': r0}
    for name in ('none', 'kron2', 'dense32'):
        t0 = time.perf_counter()
        try:
            if name == 'none': prec = lambda v: v
            elif name == 'kron2': prec, rel = kron2(Pl, A, Pr, 'xi|g'); info['kron_s3/s1'] = rel
            else: prec = dense32(Pl, A, Pr)
            torch.cuda.synchronize(); t1 = time.perf_counter()
            x, it, hist = gmres(mv, prec, rhs, xc, 1e-10, maxit=400)
            torch.cuda.synchronize(); t2 = time.perf_counter()
            info[name] = {'its': it, 'final': hist[-1], 'setup_s': round(t1 - t0, 3), 'solve_s': round(t2 - t1, 3),
                          'err_vs_lu': float(torch.linalg.vector_norm(x - sol) / torch.linalg.vector_norm(sol)),
                          'hist': [float('%.2e' % h) for h in hist[::max(1, len(hist) // 8)]]}
        except Exception as e:
            info[name] = repr(e)[:200]
        print(json.dumps(info), flush=True)
