import sys; sys.path.insert(0,'/root/repo')
import torch, paper_1912_04062_b200 as sk, skewgen
for n in [66, 130, 300]:
    A = torch.from_numpy(skewgen.random_skew(n, 66)).cuda()
    try:
        lam, zr, zi = sk.skew_eig(A)
        print(n, "ok", float(lam[0]))
    except Exception as ex:
        print(n, "ERR", ex)
