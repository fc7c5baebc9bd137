"""Diagnostics for the parity gates (GPU): (1) one bf16 Linear(+ReLU) op on
identical inputs, its outputs against float64 numpy; (2) forward drift of a
network's end-to-end forward against the oracle's own forward, op by op."""
import sys
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_1912_01703_b200 as be  # noqa: E402
import synth  # noqa: E402
from oracle import nets as onets  # noqa: E402
from teacher import OpTrace, forward_drift  # noqa: E402


def rel(x, o):
    x, o = np.asarray(x, np.float64), np.asarray(o, np.float64)
    return float(np.abs(x - o).max() / max(np.abs(o).max(), 1e-30))


def linear_probe(B, IN, OUT, act, xrelu):
    be.set_compute_dtype("bf16")
    rng = np.random.default_rng(0)
    x = synth.bf16_values(rng.standard_normal((B, IN)))
    if xrelu:
        x = np.maximum(x, 0)
    W = (rng.standard_normal((IN, OUT)) / np.sqrt(IN)).astype(np.float32)
    b = (rng.standard_normal(OUT) / np.sqrt(IN)).astype(np.float32)
    g = synth.bf16_values(rng.standard_normal((B, OUT)) * 1e-3)
    xl = be.tensor(x, requires_grad=True)
    Wl = be.tensor(W, requires_grad=True)
    bl = be.tensor(b, requires_grad=True)
    y = be.linear(be.cast(xl, "bf16"), Wl, bl, act=act)
    y.backward(be.tensor(g, dtype="bf16"))
    yd = y.numpy().astype(np.float64)
    Wb = synth.bf16_values(W).astype(np.float64)
    z = x.astype(np.float64) @ Wb + b
    mask = (yd > 0) if act else np.ones_like(yd, bool)
    dz = g.astype(np.float64) * mask
    print(f"B={B} IN={IN} OUT={OUT} act={act} xrelu={xrelu}: "
          f"y {rel(yd, np.maximum(z, 0) if act else z):.2e}  "
          f"dW {rel(Wl.grad.numpy(), x.T.astype(np.float64) @ dz):.2e}  "
          f"db {rel(bl.grad.numpy(), dz.sum(0)):.2e}  "
          f"dx(Wbf16) {rel(xl.grad.numpy(), dz @ Wb.T):.2e}  dx(W) {rel(xl.grad.numpy(), dz @ W.T.astype(np.float64)):.2e}"
          f"  mask-vs-ref {int(((yd > 0) != (z > 0)).sum()) if act else 0}")


def drift(name, dtype):
    be.set_compute_dtype(dtype)
    if name in ("vgg19", "mobilenetv2"):
        seed = 25 if name == "vgg19" else 26
        onet = onets.VGG19(seed=seed) if name == "vgg19" else onets.MobileNetV2(seed=seed)
        pnet = be.nn.VGG19(seed=seed) if name == "vgg19" else be.nn.MobileNetV2(seed=seed)
        x = synth.normal((2, 3, 224, 224), seed, 1)
        x = synth.bf16_values(x) if dtype == "bf16" else x
        batch = (be.nn.images_to_device(x, dtype), be.tensor(synth.labels(2, 1000, seed)))
    elif name == "resnet50":
        onet, pnet = onets.ResNet50(), be.nn.ResNet50()
        x = synth.normal((2, 3, 224, 224), 21, 1)
        x = synth.bf16_values(x) if dtype == "bf16" else x
        batch = (be.nn.images_to_device(x, dtype), be.tensor(synth.labels(2, 1000, 21)))
        seed = 21
    else:
        sizes = (4096, 4096, 4096, 1000)
        onet, pnet = onets.MLP(sizes), be.nn.MLP(sizes)
        x = synth.bf16_values(synth.normal((1024, 4096), 24, 1))
        batch = (be.tensor(x, dtype=dtype), be.tensor(synth.labels(1024, 1000, 24)))
        seed = 24
    pnet.load(synth.make_params(onet.param_specs(), seed))
    tr = OpTrace(be.api, pnet).install(be.nn)
    try:
        pnet.loss(*batch)
    finally:
        tr.uninstall(be.nn)
    for i, op, e in forward_drift(be, tr):
        print(f"  {name} {dtype} #{i:3d} {op:14s} {e:.3e}")


def repeat_probe(B, IN, OUT, reps=8):
    """Same Linear+ReLU op on identical inputs several times (the autotuner
    cycles GEMM variants over the first calls): outputs bitwise across runs,
    and each run's backward against float64 with its OWN mask."""
    be.set_compute_dtype("bf16")
    rng = np.random.default_rng(1)
    x = np.maximum(synth.bf16_values(rng.standard_normal((B, IN))), 0)
    W = (rng.standard_normal((IN, OUT)) / np.sqrt(IN)).astype(np.float32)
    b = (rng.standard_normal(OUT) / np.sqrt(IN)).astype(np.float32)
    g = synth.bf16_values(rng.standard_normal((B, OUT)) * 1e-4)
    Wl = be.tensor(W, requires_grad=True)
    bl = be.tensor(b, requires_grad=True)
    y0 = None
    for r in range(reps):
        xl = be.tensor(x, requires_grad=True)
        be.zero_grad([Wl, bl])
        y = be.linear(be.cast(xl, "bf16"), Wl, bl, act=1)
        y.backward(be.tensor(g, dtype="bf16"))
        yd = y.numpy().astype(np.float64)
        if y0 is None:
            y0 = yd
        dz = g.astype(np.float64) * (yd > 0)
        print(f"  rep {r}: y==y0 {np.array_equal(yd, y0)} signflips {int(((yd > 0) != (y0 > 0)).sum())} "
              f"maxdiff {np.abs(yd - y0).max():.2e}  dW {rel(Wl.grad.numpy(), x.T.astype(np.float64) @ dz):.2e} "
              f"db {rel(bl.grad.numpy(), dz.sum(0)):.2e}")


if __name__ == "__main__":
    be.init(0)
    if len(sys.argv) > 2:
        drift(sys.argv[1], sys.argv[2])
        sys.exit(0)
    for args in [(1024, 4096, 4096, 1, True), (1024, 4096, 4096, 0, True), (1024, 4096, 4096, 1, False),
                 (96, 384, 128, 1, False), (96, 256, 384, 1, False)]:
        linear_probe(*args)
    repeat_probe(1024, 4096, 4096)
    repeat_probe(96, 384, 128)
