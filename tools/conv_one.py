"""Run one bf16 conv shape fwd + bwd a few times (for ncu captures / timing).
usage: python tools/conv_one.py N H W C K R stride pad [iters]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1912_01703_b200 as be  # noqa: E402

N, H, W, C, K, R, st, pd = [int(v) for v in sys.argv[1:9]]
iters = int(sys.argv[9]) if len(sys.argv) > 9 else 5
be.init(0)
be.set_compute_dtype("bf16")
rng = np.random.default_rng(0)
xg = C % 64 == 0
x0 = be.tensor(rng.standard_normal((N, H, W, C)).astype(np.float32), requires_grad=xg, dtype=None if xg else "bf16")
w = be.tensor((rng.standard_normal((K, R, R, C)) / np.sqrt(C * R * R)).astype(np.float32), requires_grad=True)
P = (H + 2 * pd - R) // st + 1
Q = (W + 2 * pd - R) // st + 1
g = be.tensor(rng.standard_normal((N, P, Q, K)).astype(np.float32), dtype="bf16")
for i in range(iters):
    be.synchronize()
    t0 = time.perf_counter()
    x = be.cast(x0, "bf16") if xg else x0
    y = be.conv2d(x, w, None, st, pd)
    y.backward(g)
    be.synchronize()
    print(f"iter {i}: {(time.perf_counter() - t0) * 1e3:.3f} ms fwd+bwd", flush=True)
