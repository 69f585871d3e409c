import sys, os
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_2001_04109_b200 as fs
p, n, k = 131071, 4096, 4096
f = fs.PrimeField(p)
a = fs.random_matrix(f, n, k, 42)
ad = torch.from_numpy(a.view(np.int64)).cuda()
cd = torch.zeros((n, n), dtype=torch.int64, device='cuda')
pol = fs.RecursionPolicy(1024, fs.UNLIMITED_LEVELS)
s = torch.cuda.current_stream().cuda_stream
for i in range(4):
    if i == 3: print("---- traced step", file=sys.stderr)
    fs.syrk_dev(p, 1, ad.data_ptr(), n, k, k, 0, cd.data_ptr(), n, pol, False, s)
    torch.cuda.synchronize()
