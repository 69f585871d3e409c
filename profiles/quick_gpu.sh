timeout 60 python -c "
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, paper_2001_04109_b200 as fs, oracle_py as orc
for p in (131071, 2147483647, 65521, 65537):
    f=fs.PrimeField(p)
    for (m,n,k) in ((1,1,1),(300,129,1000),(256,256,256)):
        a=orc.random_matrix(p,m,k,1); b=orc.random_matrix(p,n,k,2)
        c=fs.gemm_nt(f,a,b)
        s=orc.syrk_classical(p,np.vstack([a,b]))
        print(p,m,n,k,np.array_equal(c, s[m:,:m].T))
"
echo rc=$?
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
