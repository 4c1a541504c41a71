"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs /root/reference to compile oracle/_ref):
    python tests/golden/make_golden.py
The fixtures pin the C restatement (oracle/rutv_oracle.c) without the
reference present, and they are the known-answer vectors the GPU parity tests
compare against.  Sizes are small on purpose (the whole set is < 2 MB).
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (name, m, n, b, q, seedA, seedG, kind) -- shapes from test_randutv_blocked.cpp:83-88
# and acceptance.cpp:96-99 plus ragged final blocks like every BASELINE config.
RANDUTV_CASES = [
    ("r24_b8_q1", 24, 24, 8, 1, 300 + 24 * 31 + 24, 7, "gaussian"),
    ("r25_b8_q1", 25, 25, 8, 1, 300 + 25 * 31 + 25, 7, "gaussian"),
    ("r16_b4_q0", 16, 16, 4, 0, 300 + 16 * 31 + 16, 7, "gaussian"),
    ("r6_b8_q1", 6, 6, 8, 1, 300 + 6 * 31 + 6, 7, "gaussian"),
    ("r64_b16_q2", 64, 64, 16, 2, 1000, 1001, "gaussian"),
    ("r100_b32_q1", 100, 100, 32, 1, 1002, 1003, "gaussian"),
    ("r130_b48_q0", 130, 130, 48, 0, 1004, 1005, "gaussian"),
    ("geo200_b20_q2", 200, 200, 20, 2, 9000, 0, "geometric:0.8"),
    ("diag4_b2_q2", 4, 4, 2, 2, 0, 5, "diag4321"),
    ("rect30x20_b8_q0", 30, 20, 8, 0, 300 + 30 * 31 + 20, 7, "gaussian"),
    ("rect20x30_b8_q2", 20, 30, 8, 2, 300 + 20 * 31 + 30, 7, "gaussian"),
]


def make_a(kind, m, n, seed):
    if kind == "gaussian":
        return oracle.gaussian_matrix(m, n, seed, impl="ref")
    if kind.startswith("geometric:"):
        return oracle.geometric_matrix(m, n, float(kind.split(":")[1]), seed, impl="ref")
    if kind == "diag4321":
        return np.diag([4.0, 3.0, 2.0, 1.0])
    raise ValueError(kind)


def main() -> None:
    if not oracle.available("ref"):
        raise SystemExit("oracle/_ref not buildable here (needs /root/reference)")
    # RNG: position-addressable stream (rng.cpp:29-53)
    np.savez_compressed(
        os.path.join(OUT, "rng.npz"),
        seed42_pos0=oracle.normal_stream(42, 0, 64, impl="ref"),
        seed7_pos1e9=oracle.normal_stream(7, 10**9, 64, impl="ref"),
        seed0_pos0=oracle.normal_stream(0, 0, 64, impl="ref"),
    )
    # Householder (householder.cpp:20-97)
    hq = {}
    for name, a in [("g9x4", oracle.gaussian_matrix(9, 4, 70, impl="ref")),
                    ("g40x12", oracle.gaussian_matrix(40, 12, 71, impl="ref")),
                    ("tri4", np.triu(np.add.outer(np.arange(4), np.arange(4)) + 1.0)),
                    ("neghead3", np.diag([-2.0, 1.0, 1.0])),
                    ("zero_col5x3", np.array([[0, 1, 0], [0, 0, 0], [0, 0, 0], [0, 0, 0], [0, 0, 0]], float))]:
        qr, tau, twy = oracle.hqr(a, impl="ref")
        hq[name + "_a"], hq[name + "_qr"], hq[name + "_tau"], hq[name + "_twy"] = a, qr, tau, twy
    np.savez_compressed(os.path.join(OUT, "hqr.npz"), **hq)
    # Jacobi (jacobi_svd.cpp:39-148); 2x2 known answer sqrt(45), sqrt(5)
    sv = {}
    for name, a in [("k2x2", np.array([[3.0, 0.0], [4.0, 5.0]])),
                    ("g6", oracle.gaussian_matrix(6, 6, 210, impl="ref")),
                    ("g16", oracle.gaussian_matrix(16, 16, 216, impl="ref")),
                    ("shuffled_diag4", np.diag([2.0, 4.0, 1.0, 3.0])),
                    ("rank1_5", np.outer(oracle.gaussian_matrix(5, 1, 220, impl="ref"),
                                         oracle.gaussian_matrix(5, 1, 221, impl="ref")))]:
        u, s, v = oracle.svd_block(a, impl="ref")
        sv[name + "_a"], sv[name + "_u"], sv[name + "_s"], sv[name + "_v"] = a, u, s, v
    np.savez_compressed(os.path.join(OUT, "svd.npz"), **sv)
    # gemm (gemm.cpp:21-75), all transpose combinations
    gm = {}
    a = oracle.gaussian_matrix(5, 4, 11, impl="ref")
    b = oracle.gaussian_matrix(4, 3, 12, impl="ref")
    c0 = oracle.gaussian_matrix(5, 3, 10, impl="ref")
    gm["a"], gm["b"], gm["c0"] = a, b, c0
    for ta in (0, 1):
        for tb in (0, 1):
            aa = a.T.copy() if ta else a
            bb = b.T.copy() if tb else b
            gm[f"c_{ta}{tb}"] = oracle.gemm(-0.75, ta, aa, tb, bb, 0.5, c0, impl="ref")
    np.savez_compressed(os.path.join(OUT, "gemm.npz"), **gm)
    # randUTV end to end (randutv_blocked.cpp:84-157)
    for name, m, n, b, q, sa, sg, kind in RANDUTV_CASES:
        a = make_a(kind, m, n, sa)
        t, u, v = oracle.randutv(a, b=b, q=q, seed=sg, impl="ref")
        np.savez_compressed(os.path.join(OUT, f"randutv_{name}.npz"), a=a, t=t, u=u, v=v,
                            meta=np.array([m, n, b, q, sg], dtype=np.int64))
    # .rutv files written by the reference (matrix_io.cpp:40-50) + lowrank_error values
    # (metrics.cpp:32-46) for the r64 factorization, Frobenius and spectral
    oracle.ref_write_rutv(os.path.join(OUT, "g5x3.rutv"), oracle.gaussian_matrix(5, 3, 77, impl="ref"))
    oracle.ref_write_rutv(os.path.join(OUT, "empty0x4.rutv"), np.zeros((0, 4)))
    r = np.load(os.path.join(OUT, "randutv_r64_b16_q2.npz"))
    ks = np.array([0, 1, 8, 16, 33, 63, 64])
    np.savez_compressed(os.path.join(OUT, "lowrank_r64.npz"), ks=ks,
                        fro=np.array([oracle.ref_lowrank_error(r["a"], r["t"], r["u"], r["v"], k) for k in ks]),
                        spec=np.array([oracle.ref_lowrank_error(r["a"], r["t"], r["u"], r["v"], k, "spec")
                                       for k in ks]))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
