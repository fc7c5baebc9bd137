"""Time the stem convolution kernel alone (CUDA events via be.prof_*).
usage: python tools/stem_probe.py [N H W K R stride pad]"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1912_01703_b200 as be  # noqa: E402

N, H, W, K, R, st, pd = [int(v) for v in sys.argv[1:8]] if len(sys.argv) > 7 else (256, 224, 224, 64, 7, 2, 3)
be.init(0)
be.set_compute_dtype("bf16")
rng = np.random.default_rng(0)
x = be.tensor(rng.standard_normal((N, H, W, 8)).astype(np.float32), dtype="bf16")
w = be.tensor((rng.standard_normal((K, R, R, 8)) / np.sqrt(8 * R * R)).astype(np.float32), dtype="bf16")
with be.no_grad():
    for _ in range(3):
        be.conv2d(x, w, None, st, pd)
    be.synchronize()
    be.prof_enable(True)
    for _ in range(10):
        be.conv2d(x, w, None, st, pd)
    be.synchronize()
    be.prof_enable(False)
recs = [r for r in be.prof_read() if r["name"].startswith("conv")]
ts = sorted(1e3 * r["ms"] for r in recs)
print(f"{recs[0]['name']} {recs[0]['m']}x{recs[0]['n']}x{recs[0]['k']}: median {ts[len(ts) // 2]:.1f} us "
      f"({recs[0]['flops'] / (ts[len(ts) // 2] * 1e-6) / 1e12:.0f} TF/s)")
