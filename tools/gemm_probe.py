"""Run one GEMM shape a few times (for ncu captures / quick timing).
usage: python tools/gemm_probe.py M N K ta tb [reps]"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1912_01703_b200 as be  # noqa: E402

M, N, K, ta, tb = map(int, sys.argv[1:6])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 10
be.init(0)
rng = np.random.default_rng(0)
A = be.tensor(rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32), dtype="bf16")
B = be.tensor(rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32), dtype="bf16")
D = be.empty((M, N), "bf16")
for _ in range(40):  # autotune settles
    be.gemm(A, B, D, trans_a=bool(ta), trans_b=bool(tb))
be.synchronize()
be.prof_read()
be.prof_enable(True)
for _ in range(reps):
    be.gemm(A, B, D, trans_a=bool(ta), trans_b=bool(tb))
be.prof_enable(False)
recs = be.prof_read()
ms = sorted(r["ms"] for r in recs)[len(recs) // 2]
print(f"{recs[0]['name']:16s} {M}x{N}x{K} ta={ta} tb={tb}: {ms * 1e3:8.1f} us  {2 * M * N * K / ms / 1e9:7.1f} TFLOP/s "
      f"{2 * (M * K + N * K + M * N) / ms / 1e6:7.1f} GB/s", flush=True)
