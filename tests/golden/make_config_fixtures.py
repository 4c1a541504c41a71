"""Reference fixtures for the BASELINE configs the oracle cannot finish inside a test.

TEST INFRASTRUCTURE.  Run once in the build container (needs oracle/_ref, i.e.
/root/reference); the outputs are committed under tests/golden/ and the GPU
tests (tests/test_gpu_configs.py) compare against them on the B200 box, where
/root/reference does not exist:

    python tests/golden/make_config_fixtures.py config2   # ~15 min (1 core for the reference)
    python tests/golden/make_config_fixtures.py config3   # ~5 min

config2  n=4000, A = geometric_matrix(n, n, 10^(-12/3999), seedA=1) (metrics.cpp:95-110),
         b=128, q=2, G = RngState(seedG=2) (rng.cpp:29-53): the UNMODIFIED reference
         randutv() (randutv_blocked.cpp:84-157) run to completion.  Stored: diag(T), a fixed
         sample of upper-triangle T entries, U / V at a fixed row sample for every column,
         the reference's own invariants (residual, orthogonality in three norms) and a
         SHA-256 of A's bytes (the test regenerates A with the C port and checks the hash,
         so both sides factor bit-identical input).
config4shape  the same first-step fixture at config 4's n = 30000, b = 256, q = 2 (Gaussian A:
         config 4's cliff matrix comes from the GPU Haar generator); ~40 min on one core.
config3  n=10000 Gaussian A (metrics.cpp:90-93, seedA=1), b=256, q=1, seedG=2: the reference's
         state after its FIRST step through the public step API (ref_randutv_steps, the
         randutv() loop replayed on build_v_alpha / apply_q_right / build_u_alpha /
         apply_qt_left / beta_stage, randutv_blocked.hpp:39-72 -- bit-identical to randutv()
         when run to completion, tests/test_oracle_pin.py).

A is generated with the C restatement (oracle.geometric_matrix / gaussian_matrix, OpenMP
over independent columns, bit-identical to the reference -- pinned in
tests/test_oracle_pin.py); `--verify-a` additionally regenerates it with the reference
itself and asserts byte equality before factoring.
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
EPS = np.finfo(np.float64).eps


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.asfortranarray(a).tobytes(order="F")).hexdigest()


def spec2(q: np.ndarray) -> float:
    """||Q'Q - I||_2 (symmetric: largest |eigenvalue|)."""
    e = q.T @ q - np.eye(q.shape[1])
    w = np.linalg.eigvalsh(e)
    return float(np.max(np.abs(w)))


def invariants(a, t, u, v) -> dict:
    nf = np.linalg.norm(a)
    out = {"resid_fro": float(np.linalg.norm(a - u @ t @ v.T) / nf)}
    for name, q in (("u", u), ("v", v)):
        e = q.T @ q - np.eye(q.shape[1])
        out[f"orth_{name}_fro"] = float(np.linalg.norm(e))
        out[f"orth_{name}_max"] = float(np.max(np.abs(e)))
        out[f"orth_{name}_spec"] = spec2(q)
    return out


def config2(verify_a: bool) -> None:
    n, b, q, seed_a, seed_g = 4000, 128, 2, 1, 2
    beta = 10 ** (-12 / (n - 1))
    t0 = time.time()
    a = oracle.geometric_matrix(n, n, beta, seed_a)
    print(f"A (port, OpenMP) {time.time() - t0:.1f} s", flush=True)
    if verify_a:
        t0 = time.time()
        ar = oracle.geometric_matrix(n, n, beta, seed_a, impl="ref")
        assert np.array_equal(a, ar), "port geometric_matrix differs from the reference"
        print(f"A (reference) {time.time() - t0:.1f} s: identical", flush=True)
        del ar
    t0 = time.time()
    t, u, v = oracle.randutv(a, b=b, q=q, seed=seed_g, impl="ref")
    dt = time.time() - t0
    print(f"reference randutv {dt:.1f} s", flush=True)
    rng = np.random.default_rng(20261020)
    ii = rng.integers(0, n, 40000)
    jj = rng.integers(0, n, 40000)
    keep = ii <= jj
    ii, jj = ii[keep], jj[keep]
    rows = np.sort(rng.choice(n, 96, replace=False))
    inv = invariants(a, t, u, v)
    print(inv, flush=True)
    np.savez_compressed(
        os.path.join(OUT, "config2_ref.npz"),
        n=n, b=b, q=q, seed_a=seed_a, seed_g=seed_g, beta=beta, a_sha256=sha(a),
        diag=np.diag(t).copy(), t_i=ii, t_j=jj, t_val=t[ii, jj], rows=rows,
        u_rows=u[rows, :], v_rows=v[rows, :], ref_seconds=dt,
        **{f"ref_{k}": val for k, val in inv.items()})


def config3(n=10000, b=256, q=1, name="config3_step1_ref.npz") -> None:
    seed_a, seed_g = 1, 2
    t0 = time.time()
    a = oracle.gaussian_matrix(n, n, seed_a)
    print(f"A {time.time() - t0:.1f} s", flush=True)
    t0 = time.time()
    t, u, v = oracle.randutv(a, b=b, q=q, seed=seed_g, max_steps=1, impl="ref")
    dt = time.time() - t0
    print(f"reference first step {dt:.1f} s", flush=True)
    rng = np.random.default_rng(20261021)
    cols = np.sort(rng.choice(np.arange(b, n), 160, replace=False))
    rows = np.sort(rng.choice(n, 96, replace=False))
    # trailing matrix T22 after the step (rows/cols >= b): depends on the full Q_v, Q_u
    ti = rng.integers(b, n, 30000)
    tj = rng.integers(b, n, 30000)
    np.savez_compressed(
        os.path.join(OUT, name),
        n=n, b=b, q=q, seed_a=seed_a, seed_g=seed_g, a_sha256=sha(a),
        diag=np.diag(t)[:b].copy(), strip_cols=cols, strip=t[:b, cols],
        rows=rows, u_rows=u[rows, :b], v_rows=v[rows, :b],
        t22_i=ti, t22_j=tj, t22_val=t[ti, tj], a_fro=float(np.linalg.norm(a)), ref_seconds=dt)


if __name__ == "__main__":
    if not oracle.available("ref"):
        raise SystemExit("oracle/_ref not buildable here (needs /root/reference)")
    what = sys.argv[1:] or ["config2", "config3"]
    if "config3" in what:
        config3()
    if "config4shape" in what:  # config 4's n, b, q on a Gaussian A (its cliff A needs the GPU generator)
        config3(30000, 256, 2, "config4shape_step1_ref.npz")
    if "config2" in what:
        config2("--verify-a" in what)
