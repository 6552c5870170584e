import sys, numpy as np, torch, faulthandler
faulthandler.dump_traceback_later(60, exit=True)
sys.path.insert(0, '/root/repo')
import paper_1912_04062_b200 as sk, skewgen
n = int(sys.argv[1])
A = skewgen.random_skew(n, n)
print("band", flush=True)
Ab, V, T, tau, npn = sk.reduce_to_band(torch.from_numpy(A).cuda()); torch.cuda.synchronize(); print("band ok", npn, flush=True)
AB = np.zeros((65, n))
for c in range(n):
    for d in range(65):
        if c + d < n: AB[d, c] = A[c + d, c]
ABt = torch.from_numpy(AB.T.copy()).cuda().t()
alpha = sk.band_to_tridiag(ABt, 64); torch.cuda.synchronize(); print("b2t ok", alpha, flush=True)
X = torch.eye(n, dtype=torch.float64, device="cuda").t().contiguous().t()
alpha = sk.band_to_tridiag(ABt, 64, X); torch.cuda.synchronize(); print("b2t+bt2 ok", flush=True)
lam, Q = sk.tridiag_eig(alpha, max(n // 2, 1)); torch.cuda.synchronize(); print("trid ok", lam, flush=True)
lam, Zr, Zi = sk.skew_eig(torch.from_numpy(A).cuda()); torch.cuda.synchronize(); print("full ok", lam, flush=True)
