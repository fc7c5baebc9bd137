"""Time the GEMM kernel on given shapes (CUDA events via be_prof)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1912_01703_b200 as be  # noqa: E402

be.init(0)
shapes = [(1024, 4096, 4096, 0, 0), (4096, 4096, 1024, 1, 0), (1024, 4096, 1000, 0, 1), (1024, 1000, 4096, 0, 0),
          (8192, 8192, 8192, 0, 1), (802816, 64, 576, 0, 1), (50176, 256, 2304, 0, 1), (200704, 128, 1152, 0, 1)]
rng = np.random.default_rng(0)
for (M, N, K, ta, tb) in shapes:
    A = be.tensor(rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32), dtype="bf16")
    B = be.tensor(rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32), dtype="bf16")
    D = be.empty((M, N), "bf16")
    for _ in range(3):
        be.gemm(A, B, D, trans_a=bool(ta), trans_b=bool(tb))
    be.synchronize()
    be.prof_read()
    be.prof_enable(True)
    for _ in range(20):
        be.gemm(A, B, D, trans_a=bool(ta), trans_b=bool(tb))
    be.prof_enable(False)
    recs = be.prof_read()
    ms = sorted(r["ms"] for r in recs)[len(recs) // 2]
    print(f"{os.environ.get('BE_GEMM_PAIR', 'auto'):>4} {recs[0]['name']:16s} {M}x{N}x{K} ta={ta} tb={tb}: "
          f"{ms * 1e3:8.1f} us  {2 * M * N * K / ms / 1e9:7.1f} TFLOP/s", flush=True)
