import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_2104_05782_b200 as rutv
for (n, b, q) in [(257, 64, 2), (257, 64, 1), (256, 64, 2), (257, 32, 2), (200, 64, 2)]:
    a = oracle.gaussian_matrix(n, n, 21)
    g = oracle.normal_stream(4, 0, oracle.stream_length(n, n, b))
    t, u, v = rutv.factorize(a, b=b, q=q, seed=4, g=g)
    tr, ur, vr = oracle.randutv(a, b=b, q=q, seed=4)
    dg, dr = np.diag(t), np.diag(tr)
    rel = np.abs(dg - dr) / np.abs(dr)
    print(n, b, q, "single-gpu diag rel max", rel.max(), "argmax", rel.argmax(), "tail", dr[-3:])
