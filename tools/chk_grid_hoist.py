import os, sys
sys.path.insert(0, '/root/repo') if os.path.exists('/root/repo') else None
import numpy as np, oracle, paper_2104_05782_b200 as rutv
from tests._util import compare_to_oracle
n,b,q=520,128,2
a=oracle.gaussian_matrix(n,n,77+n)
g=oracle.normal_stream(3,0,oracle.stream_length(n,n,b))
ref=oracle.randutv(a,b=b,q=q,seed=3)
for tag,kw in [("native",{}),("grid22",dict(grid=(2,2),grid_sim=True)),("grid11",dict(grid=(1,2),grid_sim=True))]:
    got=rutv.factorize(a,b=b,q=q,seed=3,g=g,**kw)
    try:
        out=compare_to_oracle(a,got,ref,t_tol=1,uv_tol=1,diag_rel=1)
    except AssertionError as e:
        out=str(e)
    print(tag, os.environ.get("RUTV_HOIST","1"), out)
