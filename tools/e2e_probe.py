"""Probe the end-to-end C2 loop: device-only vs pipelined H2D vs serial H2D."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1912_01703_b200 as be  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
stream = torch.cuda.Stream(priority=-1)  # compute stream outranks the side streams
be.init(0, stream.cuda_stream)
be.set_compute_dtype(cfg["dtype"])
model = bench.make_model(cfg, be)
hb = bench.host_batch(cfg, 1)
dts = ["bf16" if (i == 0 and cfg["net"] != "ncf" and cfg["dtype"] == "bf16") else None for i in range(len(hb))]
shapes = [(a.shape, d or {np.dtype(np.int32): "i32", np.dtype(np.float32): "f32"}[a.dtype]) for a, d in zip(hb, dts)]
pinned = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in hb]
host = [(p.data_ptr(), p.numel() * p.element_size()) for p in pinned]
pipe = be.api.InputPipeline(shapes)
loss_host = torch.empty(1, dtype=torch.float32).pin_memory()


def step(b):
    return be.nn.train_step(model, b, lr=0.01, momentum=0.9, weight_decay=1e-4)


def run(mode, n=30):
    be.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    if mode == "pipe":
        pipe.put(0, host)
    for i in range(n):
        cur = i % 2
        if mode == "device":
            loss = step(pipe.bufs[0])
        elif mode == "pipe":
            loss = step(pipe.get(cur))
            pipe.release(cur)
            if i + 1 < n:
                pipe.put(1 - cur, host)
        else:
            for t, (ptr, nb) in zip(pipe.bufs[0], host):
                be.api.copy_from_host_on(t, ptr, nb, 0)
            loss = step(pipe.bufs[0])
        if mode != "device":
            be.api.call("be_tensor_copy_to_host_async", loss.handle, C.c_void_p(loss_host.data_ptr()), 4)
    t_enq = time.perf_counter() - t0
    e1.record(stream)
    be.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{mode:7s} {ms:.4f} ms/step  ({cfg['batch'] / ms * 1e3:,.0f} samples/s)  host enqueue {t_enq / n * 1e3:.4f} ms/step")


for _ in range(5):
    step(pipe.bufs[0])
for mode in ["device", "pipe", "serial", "device", "pipe"]:
    run(mode)
