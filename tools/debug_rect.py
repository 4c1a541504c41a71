import sys, numpy as np
sys.path.insert(0, '/root/repo')
import oracle, paper_2104_05782_b200 as rutv
m, n, b, q = 20, 30, 8, 2
a = oracle.gaussian_matrix(m, n, 300 + 31 * m + n)
g = oracle.normal_stream(7, 0, oracle.stream_length(m, n, b))
tg, ug, vg = rutv.factorize(a, b=b, q=q, seed=7, g=g)
tr, ur, vr = oracle.randutv(a, b=b, q=q, seed=7)
np.set_printoptions(precision=3, linewidth=200, suppress=True)
dv = np.sign(np.einsum("ij,ij->j", vg, vr))
print("V col maxdiff", np.max(np.abs(vg - vr * dv), axis=0))
print("T diff rows", np.max(np.abs(tg - tr), axis=1))
print("resid", np.linalg.norm(a - ug @ tg @ vg.T), np.linalg.norm(a - ur @ tr @ vr.T))
print("orth", np.linalg.norm(vg.T @ vg - np.eye(n)), np.linalg.norm(vr.T @ vr - np.eye(n)))
for k in (1, 2, 3):
    tg, ug, vg = rutv.factorize(a, b=b, q=q, seed=7, g=g, max_steps=k)
    tr, ur, vr = oracle.randutv(a, b=b, q=q, seed=7, max_steps=k)
    dv = np.sign(np.einsum("ij,ij->j", vg, vr)); dv[dv==0]=1
    print(k, "V col maxdiff", np.max(np.abs(vg - vr * dv), axis=0))
