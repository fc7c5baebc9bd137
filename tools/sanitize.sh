#!/bin/bash
# compute-sanitizer passes over small invocations of the hot path (1 GPU),
# and the parity suites with allocator poisoning (BE_ALLOC_POISON=1: every
# block handed out is filled with 0xFF bytes = NaN, so a kernel that reads
# memory it did not write shows up as a parity failure).
# usage: tools/sanitize.sh r02   → gpurun_out/<tag>_sanitize_*.txt
T=${1:-r02}
mkdir -p gpurun_out
CS=compute-sanitizer
SMALL='import sys; sys.path[:0]=[".", "tests"]
import numpy as np, paper_1912_01703_b200 as be, synth
from oracle import nets as onets
be.init(0); be.set_compute_dtype("bf16")
for net, shape in [(be.nn.ResNet50(layers=(1,1,1,1), base=16, classes=10), (4,3,64,64)),
                   (be.nn.MobileNetV2(classes=10, width=0.5, settings=((1,16,1,1),(6,24,2,2))), (4,3,32,32)),
                   (be.nn.VGG19(classes=10, width=1/8, image=32), (4,3,32,32))]:
    net.load(synth.make_params(net.param_specs(), 0))
    x = be.nn.images_to_device(synth.normal(shape, 0, 1), "bf16"); y = be.tensor(synth.labels(shape[0], 10, 0))
    for _ in range(2):
        be.nn.train_step(net, (x, y), lr=0.01, momentum=0.9, weight_decay=1e-4, overlap_sgd=True)
    be.synchronize()
u, i, l = synth.ncf_batch(512, 300, 200, 0)
n = be.nn.NCF(n_users=300, n_items=200).load(synth.make_params(onets.NCF(n_users=300, n_items=200).param_specs(), 0))
for _ in range(2):
    be.nn.train_step(n, (be.tensor(u), be.tensor(i), be.tensor(l)), lr=0.01, momentum=0.9, overlap_sgd=True, sparse_embeddings=True)
be.synchronize(); print("ok")'
timeout 1500 $CS --tool memcheck --leak-check no --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_sanitize_memcheck_smoke.txt 2>&1
timeout 1500 $CS --tool memcheck --print-limit 20 python -c "$SMALL" > gpurun_out/${T}_sanitize_memcheck_nets.txt 2>&1
timeout 1500 $CS --tool synccheck --print-limit 20 python -c "$SMALL" > gpurun_out/${T}_sanitize_synccheck_nets.txt 2>&1
timeout 1500 $CS --tool racecheck --racecheck-report hazard --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_sanitize_racecheck_smoke.txt 2>&1
BE_ALLOC_POISON=1 timeout 1500 python -m pytest tests/test_gpu_cnn.py tests/test_gpu_mlp.py tests/test_gpu_mobile.py tests/test_gpu_sparse.py -q -x > gpurun_out/${T}_sanitize_poison.txt 2>&1
for f in gpurun_out/${T}_sanitize_*.txt; do echo "== $f"; tail -n 4 $f; done
