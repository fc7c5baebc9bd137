"""Print the GEMM/conv/SGD launch timeline (CUDA events, all streams) of one
training step.  usage: python tools/timeline.py [c2] [overlap|fused]"""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1912_01703_b200 as be  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
mode = sys.argv[2] if len(sys.argv) > 2 else "overlap"
be.init(0)
be.set_compute_dtype(cfg["dtype"])
model = bench.make_model(cfg, be)
hb = bench.host_batch(cfg, 1)
batch = []
for i, a in enumerate(hb):
    if i == 0 and cfg["net"] != "ncf" and cfg["dtype"] == "bf16":  # bf16 bits (bench.py's dev_batch)
        t = be.empty(a.shape, "bf16")
        be.api.call("be_tensor_copy_from_host_async", t.handle, a.ctypes.data_as(__import__("ctypes").c_void_p),
                    a.nbytes)
        batch.append(t)
    else:
        batch.append(be.tensor(a))
be.synchronize()
step = lambda: be.nn.train_step(model, batch, lr=0.01, momentum=0.9, weight_decay=1e-4,  # noqa: E731
                                overlap_sgd=mode == "overlap")
for _ in range(15):
    step()
be.synchronize()
be.prof_enable(True)
for _ in range(2):
    step()
be.synchronize()
be.prof_enable(False)
recs = be.prof_read()
recs = recs[len(recs) // 2:]
base = recs[0]["t0"]
for r in sorted(recs, key=lambda r: r["t0"]):
    bw = r["bytes"] / (r["ms"] / 1e3) / 1e9 if r["ms"] else 0
    tf = r["flops"] / (r["ms"] / 1e3) / 1e12 if r["ms"] else 0
    print(f"{r['t0'] - base:8.1f} ms? {1e3 * (r['t0'] - base):9.1f} us  +{1e3 * r['ms']:7.1f} us  {r['name']:18s} "
          f"{r['m']}x{r['n']}x{r['k']}  {tf:7.1f} TF/s  {bw:7.0f} GB/s")
