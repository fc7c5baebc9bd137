"""One rank of the world-2 peer-memory data-parallel test (test infrastructure;
tests/test_gpu_p2p.py spawns two of these on ONE GPU — CUDA IPC works between
processes on the same device and the GPU time-slices their barrier kernels).
Handles are exchanged over gloo (torch.distributed, CPU); libbe itself uses
no NCCL on this path."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def main():
    rank, world, port, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    dtype, steps = sys.argv[5], int(sys.argv[6])
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    import paper_1912_01703_b200 as be
    import synth
    be.init(0)
    be.set_compute_dtype(dtype)
    sizes = (96, 136, 72, 24)
    net = be.nn.MLP(sizes)
    P = synth.make_params(net.param_specs(), 61)
    net.load(P)
    B = 64
    x = synth.normal((B, sizes[0]), 61, 1)
    y = synth.labels(B, sizes[-1], 61)
    lo, hi = rank * B // world, (rank + 1) * B // world
    xs = be.tensor(synth.bf16_values(x[lo:hi]) if dtype == "bf16" else x[lo:hi], dtype=dtype if dtype == "bf16" else None)
    ys = be.tensor(y[lo:hi])
    blob = be.p2p_attach(net.parameters(), rank, world, bucket_bytes=1 << 15)  # several buckets
    blobs = [None] * world
    dist.all_gather_object(blobs, blob)
    be.p2p_connect(blobs)
    losses = []
    for _ in range(steps):
        loss = be.nn.train_step(net, (xs, ys), lr=0.05, momentum=0.9, weight_decay=1e-4, overlap_sgd=True)
        losses.append(loss.item())
    status = be.p2p_status()
    params = {k: p.numpy().tolist() for k, p in net.params.items()}
    be.ddp_detach()
    json.dump({"status": status, "losses": losses, "params": params}, open(out, "w"))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
