"""Re-entrancy of the boundary ("re-entrant per handle").

Each call owns its streams and its stream-ordered workspace from the library's
per-device pool; kernel attributes are set once per (device, kernel) behind a
mutex.  Two host threads factoring on device 0 at the same time must each get
the bit-identical result of a serial run, and a call on a missing device must
fail with a status, not crash."""
import threading

import numpy as np
import pytest

import oracle
import paper_2104_05782_b200 as rutv

pytestmark = pytest.mark.gpu


def test_two_threads_bit_identical():
    cases = [(600, 64, 1, 11), (520, 128, 2, 12)]
    inputs = []
    for n, b, q, s in cases:
        a = oracle.gaussian_matrix(n, n, s)
        g = oracle.normal_stream(s + 1, 0, oracle.stream_length(n, n, b))
        inputs.append((a, b, q, s + 1, g))
    serial = [rutv.factorize(a, b=b, q=q, seed=s, g=g) for a, b, q, s, g in inputs]
    results = {}
    errors = []

    def worker(k):
        try:
            a, b, q, s, g = inputs[k % 2]
            results[k] = [rutv.factorize(a, b=b, q=q, seed=s, g=g) for _ in range(3)]
        except Exception as exc:  # surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for k, runs in results.items():
        for got in runs:
            for x, y in zip(got, serial[k % 2]):
                assert np.array_equal(x, y)


def test_missing_device_is_a_status_not_a_crash():
    import torch
    bad = torch.cuda.device_count()  # one past the last ordinal
    a = oracle.gaussian_matrix(40, 40, 1)
    with pytest.raises(rutv.RutvError) as ei:
        rutv.factorize(a, b=8, q=1, seed=1, device=bad)
    assert ei.value.code == 5  # RUTV_ERR_CUDA
    t, u, v = rutv.factorize(a, b=8, q=1, seed=1)  # the library is still usable
    assert np.linalg.norm(a - u @ t @ v.T) / np.linalg.norm(a) < 1e-13


def test_keep_workspace_then_release():
    """rutv_opts.keep_workspace leaves the call's workspace in the library pool (the next
    call of the same size reuses it); rutv_b200_release_workspace returns it.  Results are
    identical either way."""
    import ctypes as C
    import torch
    n, b, q = 1200, 128, 1
    a = oracle.gaussian_matrix(n, n, 21)
    ref = rutv.factorize(a, b=b, q=q, seed=5)
    o = rutv.make_opts(b=b, q=q, seed=5, keep_workspace=True)
    outs = [np.zeros((n, n), order="F") for _ in range(3)]
    st = rutv.Status()
    free0 = torch.cuda.mem_get_info()[0]
    rutv.lib().rutv_b200_factorize(C.byref(o), a.ctypes.data_as(C.c_void_p), n, n, n, None, 0,
                                   *[x for h in outs for x in (h.ctypes.data_as(C.c_void_p), n)], C.byref(st))
    rutv._raise(st)
    for x, y in zip(outs, ref):
        assert np.array_equal(x, y)
    rutv.release_workspace(0)
    assert torch.cuda.mem_get_info()[0] >= free0 - (64 << 20)  # nothing left cached beyond slack
