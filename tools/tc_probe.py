import sys, numpy as np
sys.path.insert(0, '.')
from paper_2502_16949_b200 import Engine
e = Engine(0)
rng = np.random.default_rng(0)
A = rng.uniform(-1, 1, (128, 128)).astype(np.float32)
B = rng.uniform(-1, 1, (128, 128)).astype(np.float32)
for mode in (0, 1, 2):
    for var in range(1):
        D = e.debug_tc_gemm(mode | (var << 2), A, B)
        a = A.astype(np.float64) if mode != 2 else A.T.astype(np.float64)
        b = B.astype(np.float64) if mode == 0 else B.T.astype(np.float64)
        ref = a @ b.T
        print("mode", mode, "var", var, "maxerr", float(np.abs(D - ref).max()), flush=True)
