"""On-device test-matrix generators against the reference's (metrics.cpp:90-110).

gaussian_matrix_device: A(i, j) = RngState(seed).normal_at(i + j m) (metrics.cpp:90-93).
The integer layer (splitmix word, 53-bit uniform, rng.cpp:11-27) is exact on any device,
so every value must agree with the host stream to the libm level of log / sqrt / cos /
sin (rng.cpp:29-36): a wrong counter or word would give an unrelated value.

spectrum_matrix_device: Q1 diag(sigma) Q2' with Haar Q = form_q(hqr(G)) from one
RngState (metrics.cpp:24-28, 95-110): agrees with the oracle's restatement (bit-identical
to the reference) to ||dA|| <= 1e-13 ||A||, for geometric_matrix's beta^j and for the
config-4 cliff spectrum.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2104_05782_b200 as rutv
from tests._util import to_np

pytestmark = pytest.mark.gpu


def _cm(m, n):
    return torch.empty((n, m), dtype=torch.float64, device="cuda").T


@pytest.mark.parametrize("m,n,seed", [(1000, 700, 1), (37, 53, 2**63 + 11), (1, 1, 0), (4096, 3, 42)])
def test_gaussian_matrix_matches_reference(m, n, seed):
    a = _cm(m, n)
    rutv.gaussian_matrix_device(a, seed)
    got = to_np(a)
    ref = oracle.gaussian_matrix(m, n, seed)
    rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)
    same = float(np.mean(got == ref))
    assert rel.max() <= 1e-14, rel.max()
    assert same >= 0.5, same  # most values bit-identical; the rest differ in the last bits of libm


def test_gaussian_matrix_with_leading_dimension():
    m, n = 300, 40
    full = _cm(320, n)
    full.fill_(np.nan)
    a = full[:m, :]
    rutv.gaussian_matrix_device(a, 9)
    ref = oracle.gaussian_matrix(m, n, 9)
    assert np.max(np.abs(to_np(a) - ref)) <= 1e-14 * np.max(np.abs(ref))
    assert torch.isnan(full[m:, :]).all().item()  # padding rows untouched


@pytest.mark.parametrize("m,n", [(300, 300), (257, 190), (150, 260)])
def test_geometric_matrix_matches_reference(m, n):
    beta = 10 ** (-12 / (min(m, n) - 1))
    a = _cm(m, n)
    rutv.spectrum_matrix_device(a, 5, beta=beta)
    ref = oracle.geometric_matrix(m, n, beta, 5)
    d = np.linalg.norm(to_np(a) - ref) / np.linalg.norm(ref)
    assert d <= 1e-13, d


def test_cliff_spectrum_matrix_matches_reference():
    n = 300
    i = np.arange(1, n + 1)
    sig = np.where(i <= 100, 1.0, 1e-3 * 0.999 ** (i - 100.0))  # config 4's construction, scaled
    a = _cm(n, n)
    rutv.spectrum_matrix_device(a, 3, sigma=sig)
    ref = oracle.spectrum_matrix(n, n, sig, 3)
    d = np.linalg.norm(to_np(a) - ref) / np.linalg.norm(ref)
    assert d <= 1e-13, d
    # the constructed spectrum is the one requested
    s = np.linalg.svd(to_np(a), compute_uv=False)
    assert np.max(np.abs(s - sig)) <= 1e-13


def test_generator_config_errors():
    a = _cm(10, 10)
    with pytest.raises(ValueError):
        rutv.spectrum_matrix_device(a, 1, beta=0.0)
