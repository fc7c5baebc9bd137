"""HBM-bound 1x1-conv GEMM shapes of ResNet-50 (b256): time, TF/s and the
fraction of the HBM roofline (algorithmic bytes A + B + D)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1912_01703_b200 as be  # noqa: E402

be.init(0)
shapes = [(802816, 256, 64, 0, 1), (200704, 512, 128, 0, 1), (50176, 1024, 256, 0, 1), (802816, 64, 256, 0, 1),
          (802816, 64, 64, 0, 1), (200704, 128, 512, 0, 1), (50176, 256, 1024, 0, 1), (802816, 128, 256, 0, 1)]
if len(sys.argv) > 1 and "x" in sys.argv[1]:
    shapes = [tuple(map(int, a.split("x"))) + (0, 1) for a in sys.argv[1:]]
elif len(sys.argv) > 1:
    shapes = shapes[:int(sys.argv[1])]
HBM = 6547.2e9
rng = np.random.default_rng(0)
for (M, N, K, ta, tb) in shapes:
    A = be.tensor(rng.standard_normal((M, K)).astype(np.float32), dtype="bf16")
    B = be.tensor(rng.standard_normal((N, K)).astype(np.float32), dtype="bf16")
    D = be.empty((M, N), "bf16")
    for _ in range(30):
        be.gemm(A, B, D, trans_a=bool(ta), trans_b=bool(tb))
    be.synchronize()
    be.prof_read()
    be.prof_enable(True)
    for _ in range(20):
        be.gemm(A, B, D, trans_a=bool(ta), trans_b=bool(tb))
    be.prof_enable(False)
    recs = be.prof_read()
    ms = sorted(r["ms"] for r in recs)[len(recs) // 2]
    byts = 2 * (M * K + N * K + M * N)
    print(f"{recs[0]['name']:20s} {M}x{N}x{K}: {ms * 1e3:8.1f} us  {2 * M * N * K / ms / 1e9:7.1f} TF/s  "
          f"{byts / ms / 1e6:7.1f} GB/s  hbm-frac {byts / (ms / 1e3) / HBM:.3f}", flush=True)
