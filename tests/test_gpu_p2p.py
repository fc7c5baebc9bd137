"""Peer-memory data parallelism on the B200 (-m gpu): the
fused allreduce + SGD bucket kernel (p2p.cu, be_p2p_attach / be_p2p_connect).

* world 1, in process: the kernel's update is bitwise the non-DDP overlapped
  SGD's (same sgd_elem arithmetic), over several buckets, 3 momentum steps;
* world 2, two processes sharing ONE GPU (CUDA IPC between processes on the
  same device; the GPU time-slices the two contexts' barrier kernels): after
  3 steps with momentum + wd both replicas hold bitwise identical parameters
  and match the float64 oracle's 2-replica data-parallel emulation
  (oracle/step.py: contiguous batch shards, g = mean of the shard gradients)
  at the fp32 tolerance."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import synth
from gpu_common import be_init, rel
from oracle import nets as onets
from oracle.step import train_step

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_p2p_world1_bitwise_equals_overlapped_sgd():
    be = be_init()
    be.set_compute_dtype("bf16")
    sizes = (256, 512, 384, 10)
    P = synth.make_params(onets.MLP(sizes).param_specs(), 62)
    x = be.tensor(synth.bf16_values(synth.normal((96, 256), 62, 1)), dtype="bf16")
    y = be.tensor(synth.labels(96, 10, 62))
    plain = be.nn.MLP(sizes).load(P)
    for _ in range(3):
        be.nn.train_step(plain, (x, y), lr=0.05, momentum=0.9, weight_decay=1e-4, overlap_sgd=True)
    ref = {k: p.numpy() for k, p in plain.params.items()}
    be.sgd_overlap([])
    plain._overlap = None
    net = be.nn.MLP(sizes).load(P)
    blob = be.p2p_attach(net.parameters(), 0, 1, bucket_bytes=1 << 18)  # several buckets
    be.p2p_connect([blob])
    try:
        for _ in range(3):
            be.nn.train_step(net, (x, y), lr=0.05, momentum=0.9, weight_decay=1e-4, overlap_sgd=True)
        assert be.p2p_status() == 0
        for k, p in net.params.items():
            assert np.array_equal(p.numpy(), ref[k]), k
    finally:
        be.ddp_detach()
        be.sgd_overlap([])


def test_p2p_world2_two_processes_one_gpu(tmp_path):
    be_init()
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    steps = 3
    outs = [str(tmp_path / f"r{r}.json") for r in range(2)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "p2p_worker.py"), str(r), "2", str(port), outs[r],
                               "f32", str(steps)]) for r in range(2)]
    for p in procs:
        assert p.wait(timeout=600) == 0
    res = [json.load(open(o)) for o in outs]
    assert res[0]["status"] == 0 and res[1]["status"] == 0
    for k in res[0]["params"]:
        assert np.array_equal(np.array(res[0]["params"][k]), np.array(res[1]["params"][k])), k  # replicas identical
    # oracle: 2-replica DP emulation of the same 3 steps
    sizes = (96, 136, 72, 24)
    onet = onets.MLP(sizes)
    P = synth.make_params(onet.param_specs(), 61)
    x, y = synth.normal((64, 96), 61, 1), synth.labels(64, 24, 61)
    op, bufs = dict(P), None
    for _ in range(steps):
        r = train_step(onet, op, (x, y), lr=0.05, momentum=0.9, weight_decay=1e-4, replicas=2, bufs=bufs)
        op, bufs = r["params"], r["bufs"]
    for k in op:
        assert rel(np.array(res[0]["params"][k]), op[k]) <= 1e-4, k
