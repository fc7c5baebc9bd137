"""Run N training steps of a bench config with fixed inputs and print a hash of
the loss sequence and all parameters (determinism check, e.g. BE_PDL=0 vs 1).
usage: BE_TUNE=0 python tools/det_check.py c2 [steps] [overlap|fused]"""
import hashlib
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1912_01703_b200 as be  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
mode = sys.argv[3] if len(sys.argv) > 3 else "overlap"
be.init(0)
be.set_compute_dtype(cfg["dtype"])
model = bench.make_model(cfg, be)
hb = bench.host_batch(cfg, 1)
batch = []
for i, a in enumerate(hb):
    if i == 0 and cfg["net"] != "ncf" and cfg["dtype"] == "bf16":
        t = be.empty(a.shape, "bf16")
        be.api.call("be_tensor_copy_from_host_async", t.handle, a.ctypes.data_as(__import__("ctypes").c_void_p), a.nbytes)
        batch.append(t)
    else:
        batch.append(be.tensor(a))
be.synchronize()
losses = []
for _ in range(steps):
    loss = be.nn.train_step(model, batch, lr=0.01, momentum=0.9, weight_decay=1e-4, overlap_sgd=mode == "overlap")
    losses.append(loss.item() if hasattr(loss, "item") else float(loss))
be.synchronize()
h = hashlib.sha256()
for k in sorted(model.params):
    h.update(model.params[k].numpy().tobytes())
print(sys.argv[1], mode, "losses", [repr(x) for x in losses[-2:]], "params sha256", h.hexdigest()[:16])
