"""The reference's own rounding sensitivity of diag(T) (1.1e-16 perturbation of A), q = 0 vs 2."""
import numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
for n, b, q in [(520, 128, 2), (520, 128, 0), (300, 64, 1), (256, 32, 2)]:
    a = oracle.gaussian_matrix(n, n, 77 + n)
    t = oracle.randutv(a, b=b, q=q, seed=3)[0]
    ap = np.asfortranarray(a * (1 + 1.1e-16 * np.random.default_rng(1).standard_normal(a.shape)))
    tp = oracle.randutv(ap, b=b, q=q, seed=3)[0]
    d, dp = np.diag(t), np.diag(tp)
    print(n, b, q, "diag self rel", np.max(np.abs(d - dp) / np.abs(d)), "T self", np.max(np.abs(t - tp)) / np.linalg.norm(a))
