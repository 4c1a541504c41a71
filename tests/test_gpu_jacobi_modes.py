"""Both batched Jacobi kernels against the reference's svd_block (jacobi_svd.cpp:39-148): the
column-distributed kernel (jacobi_blk.cu, default for blocks up to 512 wide) is what every other
GPU test exercises; RUTV_JACOBI=rows selects the row-distributed kernel (jacobi.cu, the only one
for wider blocks).  The switch is read once per process, hence a subprocess running the SVD
tests of test_gpu_kernels.py and one small factorization against the oracle."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

FACT = r'''
import sys
sys.path.insert(0, ".")
import numpy as np
import oracle, paper_2104_05782_b200 as rutv
from tests._util import compare_to_oracle, check_structure
n, b, q = 300, 64, 1
a = oracle.gaussian_matrix(n, n, 31)
g = oracle.normal_stream(4, 0, oracle.stream_length(n, n, b))
got = rutv.factorize(a, b=b, q=q, seed=4, g=g)
check_structure(got[0], b)
compare_to_oracle(a, got, oracle.randutv(a, b=b, q=q, seed=4))
print("ok")
'''


def test_row_distributed_kernel_still_matches():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RUTV_JACOBI="rows")
    res = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_kernels.py", "-q", "-x", "-k", "svd"], cwd=root,
                         env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    res = subprocess.run([sys.executable, "-c", FACT], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0 and "ok" in res.stdout, res.stderr[-2000:]
