"""Time one conv's backward (dgrad + wgrad) at a given geometry, bf16, through the
public API: python tools/wgrad_probe.py N C H K R stride pad [reps]
(BE_WGRAD_VARIANT=v forces the wgrad variant; be_prof records give per-kernel times)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1912_01703_b200 as be  # noqa: E402

N, C, H, K, R, st, pd = map(int, sys.argv[1:8])
reps = int(sys.argv[8]) if len(sys.argv) > 8 else 10
be.init(0)
be.set_compute_dtype("bf16")
rng = np.random.default_rng(0)
x = be.tensor(rng.standard_normal((N, H, H, C)).astype(np.float32), dtype="bf16")
w = be.tensor((rng.standard_normal((K, R, R, C)) / np.sqrt(C * R * R)).astype(np.float32), requires_grad=True)
P = (H + 2 * pd - R) // st + 1
g = be.tensor(rng.standard_normal((N, P, P, K)).astype(np.float32), dtype="bf16")
def step():
    be.zero_grad([w])
    y = be.conv2d(x, w, None, st, pd)
    y.backward(g)
for _ in range(30):
    step()
be.synchronize()
be.prof_read()
import time
be.prof_enable(True)
t0 = time.perf_counter()
for _ in range(reps):
    step()
be.synchronize()
t1 = time.perf_counter()
be.prof_enable(False)
print(f"step (fwd + wgrad only, wall) {(t1 - t0) / reps * 1e6:8.1f} us")
recs = be.prof_read()
agg = {}
for r in recs:
    agg.setdefault((r["name"], r.get("m"), r.get("n"), r.get("k")), []).append(r["ms"])
for key, v in agg.items():
    v.sort()
    print(f"{key[0]:22s} {key[1]}x{key[2]}x{key[3]}: {v[len(v) // 2] * 1e3:8.1f} us (n={len(v)})")
