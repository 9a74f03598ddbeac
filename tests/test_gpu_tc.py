"""tcgen05 (3xTF32) self test of the three operand views TransR uses."""
import numpy as np
import pytest

from paper_2502_16949_b200 import Engine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_tc_gemm_operand_views(mode):
    rng = np.random.default_rng(mode)
    A = rng.uniform(-1, 1, (128, 128)).astype(np.float32)
    B = rng.uniform(-1, 1, (128, 128)).astype(np.float32)
    eng = Engine(0)
    D = eng.debug_tc_gemm(mode, A, B)
    eng.close()
    a = A.astype(np.float64) if mode != 2 else A.T.astype(np.float64)   # a[m][k]
    b = B.astype(np.float64) if mode == 0 else B.T.astype(np.float64)   # b[n][k]
    ref = a @ b.T
    err = np.abs(D - ref).max()
    assert err < 2e-5, (mode, err, D[:2, :4], ref[:2, :4])
