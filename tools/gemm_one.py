"""Run one GEMM shape a few times (for ncu captures)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1912_01703_b200 as be
be.init(0)
M, N, K, ta, tb = [int(v) for v in sys.argv[1:6]]
rng = np.random.default_rng(0)
A = be.tensor(rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32), dtype="bf16")
B = be.tensor(rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32), dtype="bf16")
D = be.empty((M, N), "bf16")
for _ in range(5):
    be.gemm(A, B, D, trans_a=bool(ta), trans_b=bool(tb))
be.synchronize()
