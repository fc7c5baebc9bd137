"""Debug sweep of the GEMM paths (prints max rel error per config)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1912_01703_b200 as be  # noqa: E402
from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32  # noqa: E402

be.init(0)
rng = np.random.default_rng(0)


def run(dtype, ta, tb, M, N, K, exact_tf32=False):
    a = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    b = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    if dtype == "bf16" or exact_tf32:
        a = bf16_bits_to_f32(f32_to_bf16_bits(a))
        b = bf16_bits_to_f32(f32_to_bf16_bits(b))
    A, B = be.tensor(a, dtype=dtype), be.tensor(b, dtype=dtype)
    D = be.empty((M, N), "f32")
    be.gemm(A, B, D, trans_a=bool(ta), trans_b=bool(tb))
    ref = (a.T if ta else a).astype(np.float64) @ (b.T if tb else b).astype(np.float64)
    x = D.numpy()
    e = np.max(np.abs(x - ref)) / np.max(np.abs(ref))
    bad = np.argwhere(np.abs(x - ref) > 1e-3 * np.max(np.abs(ref)))
    print(f"{dtype} ta={ta} tb={tb} M={M} N={N} K={K} exact={exact_tf32}: err={e:.3e} nbad={len(bad)} "
          f"first_bad={bad[:3].tolist()} x00={x[0,0]:.4f} ref00={ref[0,0]:.4f}", flush=True)


for dtype in ["bf16", "f32"]:
    for (ta, tb) in [(0, 1), (0, 0), (1, 0), (1, 1)]:
        for (M, N, K) in [(128, 128, 64), (128, 128, 256), (256, 256, 128), (300, 200, 136)]:
            try:
                run(dtype, ta, tb, M, N, K)
            except Exception as ex:
                print("EXC", dtype, ta, tb, M, N, K, ex, flush=True)
run("f32", 0, 1, 128, 128, 32, True)
run("f32", 0, 1, 128, 128, 32, False)
