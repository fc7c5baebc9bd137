"""Per-parameter gradient error of a small bf16 ResNet vs the f64 oracle."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1912_01703_b200 as be  # noqa: E402
import synth  # noqa: E402
from oracle import nets as onets  # noqa: E402
from oracle.step import train_step  # noqa: E402
from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32  # noqa: E402

be.init(0)
dtype = sys.argv[1] if len(sys.argv) > 1 else "bf16"
base = int(sys.argv[2]) if len(sys.argv) > 2 else 16
be.set_compute_dtype(dtype)
onet = onets.ResNet50(layers=(1, 1, 1, 1), base=base, classes=10)
pnet = be.nn.ResNet50(layers=(1, 1, 1, 1), base=base, classes=10)
P = synth.make_params(onet.param_specs(), 4)
hw = int(sys.argv[3]) if len(sys.argv) > 3 else 64
bs = int(sys.argv[4]) if len(sys.argv) > 4 else 8
x = bf16_bits_to_f32(f32_to_bf16_bits(synth.normal((bs, 3, hw, hw), 4, 1)))
y = synth.labels(bs, 10, 4)
ref = train_step(onet, P, (x, y), lr=0.01)
pnet.load(P)
loss = pnet.loss(be.nn.images_to_device(x, dtype), be.tensor(y))
loss.backward()
print("loss", loss.item(), ref["loss"])
for k, p in pnet.params.items():
    g = pnet.logical(k, p.grad.numpy()).astype(np.float64)
    o = ref["grads"][k]
    fro = np.linalg.norm(g - o) / max(np.linalg.norm(o), 1e-30)
    print(f"{k:14s} fro {fro:.3e}  |g| {np.linalg.norm(g):.3e} |o| {np.linalg.norm(o):.3e}")
