"""cProfile of the host side of the eager training step (enqueue cost per step).
usage: python tools/host_profile.py [c4] [steps]"""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1912_01703_b200 as be  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
be.init(0)
be.set_compute_dtype(cfg["dtype"])
model = bench.make_model(cfg, be)
hb = bench.host_batch(cfg, 1)
batch = [be.tensor(hb[0], dtype="bf16") if cfg["dtype"] == "bf16" and cfg["net"] != "ncf" else be.tensor(hb[0])]
batch += [be.tensor(a) for a in hb[1:]]
step = lambda: be.nn.train_step(model, batch, lr=0.01, momentum=0.9, weight_decay=1e-4, overlap_sgd=True)  # noqa: E731
for _ in range(30):
    step()
be.synchronize()
import ctypes  # noqa: E402
try:  # tools/sampler.c, when LD_PRELOADed: sample the C++ side during the timed host loop
    arm = ctypes.CDLL(None).sampler_arm
except AttributeError:
    arm = lambda on: None  # noqa: E731
arm(1)
t0 = time.perf_counter()
for _ in range(steps):
    step()
t1 = time.perf_counter()
arm(0)
be.synchronize()
print(f"host enqueue {1e3 * (t1 - t0) / steps:.2f} ms/step (GPU drained after: {1e3 * (time.perf_counter() - t0) / steps:.2f})")
# one step enqueued onto an idle GPU (empty launch queue): the host's own cost
one = []
for _ in range(steps):
    be.synchronize()
    ta = time.perf_counter()
    step()
    one.append(time.perf_counter() - ta)
be.synchronize()
one.sort()
print(f"host enqueue of one step onto an idle GPU: median {1e3 * one[len(one) // 2]:.2f} ms, min {1e3 * one[0]:.2f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(steps):
    step()
pr.disable()
be.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
