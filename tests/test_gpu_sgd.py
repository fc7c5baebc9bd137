"""Parity of the optimizer configuration the bench times — SGD with momentum
0.9 and weight decay 1e-4 (DESIGN R5; oracle/optim.py) —
through all three update paths of the library, over 3 steps with momentum
buffers, against the float64 oracle (-m gpu):

* be_sgd_step (one fused multi-tensor launch after backward);
* be_sgd_overlap (each parameter updated inside backward on a side stream);
* the fused-SGD wgrad epilogue (the Linear weight update applied by the
  weight-gradient GEMM itself; no gradient is stored) at C2's 4096×4096 shape.

fp32 runs are compared end to end (3 oracle train steps) at 1e-4; the bf16
paths are compared on identical gradients (each step's device gradient fed
to the oracle's SGD; for the fused epilogue the gradient is made exactly
representable, so it is the same number on both sides)."""
import numpy as np
import pytest

import synth
from gpu_common import be_init, rel
from oracle import nets as onets
from oracle.optim import sgd_step as oracle_sgd
from oracle.step import train_step

pytestmark = pytest.mark.gpu

LR, MU, WD = 0.05, 0.9, 1e-4


def test_momentum_wd_three_steps_fp32_end_to_end():
    """fp32 (3xTF32): 3 training steps of an MLP with μ=0.9, wd=1e-4 through
    be_sgd_step vs 3 oracle steps (momentum buffers carried): loss, params and
    momentum buffers at 1e-4 after every step."""
    be = be_init()
    be.set_compute_dtype("f32")
    onet, pnet = onets.MLP((96, 136, 24)), be.nn.MLP((96, 136, 24))
    x, y = synth.normal((37, 96), 31, 1), synth.labels(37, 24, 31)
    ob, db = (x, y), (be.tensor(x), be.tensor(y))
    P = synth.make_params(onet.param_specs(), 33)
    pnet.load(P)
    params = pnet.parameters()
    op, bufs = dict(P), None
    for step in range(3):
        ref = train_step(onet, op, ob, lr=LR, momentum=MU, weight_decay=WD, bufs=bufs)
        op, bufs = ref["params"], ref["bufs"]
        be.zero_grad(params)
        loss = pnet.loss(*db)
        loss.backward()
        be.sgd_step(params, LR, MU, WD)
        assert rel(np.array(loss.item()), np.array(ref["loss"])) < 1e-4, step
        for k, p in pnet.params.items():
            assert rel(pnet.logical(k, p.numpy()), op[k]) < 1e-4, (step, k)
            v = be.sgd_momentum(p)
            assert rel(pnet.logical(k, v.numpy()), bufs[k]) < 1e-4, (step, "v", k)


@pytest.mark.parametrize("overlap", [False, True])
def test_momentum_wd_three_steps_fp32_resnet(overlap):
    """fp32 (3xTF32) ResNet (every parameter kind: KRSC conv weights with the
    stem's zero pad channels, BN γ/β, the fc head), μ=0.9, wd=1e-4, 3 steps,
    through be_sgd_step and be_sgd_overlap.  A 3-step trajectory of a
    batch-4 BN net is too ill-conditioned to compare end to end at 1e-4
    (tests/conditioning.py), so each step is checked from the device's own
    state: the loss against an oracle step from the same parameters (1e-4),
    and the update of every parameter and momentum buffer against the
    oracle's SGD fed the device's gradient (1e-6)."""
    be = be_init()
    be.set_compute_dtype("f32")
    onet = onets.ResNet50(layers=(1, 1, 1, 1), base=8, classes=10)
    pnet = be.nn.ResNet50(layers=(1, 1, 1, 1), base=8, classes=10)
    x, y = synth.normal((4, 3, 64, 64), 32, 1), synth.labels(4, 10, 32)
    ob, db = (x, y), (be.nn.images_to_device(x, "f32"), be.tensor(y))
    pnet.load(synth.make_params(onet.param_specs(), 33))
    params = pnet.parameters()
    if overlap:
        be.sgd_overlap(params, LR, MU, WD)
    try:
        for step in range(3):
            before = {k: pnet.logical(k, p.numpy()).astype(np.float64) for k, p in pnet.params.items()}
            vb = {k: be.sgd_momentum(p) for k, p in pnet.params.items()}
            vb = {k: pnet.logical(k, v.numpy()).astype(np.float64) for k, v in vb.items() if v is not None}
            ref = train_step(onet, before, ob, lr=LR)
            be.zero_grad(params)
            loss = pnet.loss(*db)
            loss.backward()
            if not overlap:
                be.sgd_step(params, LR, MU, WD)
            assert rel(np.array(loss.item()), np.array(ref["loss"])) < 1e-4, step
            for k, p in pnet.params.items():
                assert p.grad is not None, k
                g = {k: pnet.logical(k, p.grad.numpy()).astype(np.float64)}
                newp, newb = oracle_sgd({k: before[k]}, g, LR, MU, WD, {k: vb[k]} if k in vb else None)
                assert rel(pnet.logical(k, p.numpy()), newp[k]) < 1e-6, (step, k)
                assert rel(pnet.logical(k, be.sgd_momentum(p).numpy()), newb[k]) < 1e-6, (step, "v", k)
    finally:
        be.sgd_overlap([])


@pytest.mark.parametrize("overlap", [False, True])
def test_momentum_wd_identical_gradients_bf16(overlap):
    """bf16 mixed precision, μ=0.9, wd=1e-4: each step's update of the fp32
    masters and momentum buffers vs the oracle's SGD fed the SAME gradient
    (the device's), for be_sgd_step and for be_sgd_overlap (biases and the
    small head take the side-stream kernel; the 2-D weights with one wgrad
    contribution take the fused epilogue — checked separately below)."""
    be = be_init()
    be.set_compute_dtype("bf16")
    sizes = (512, 1024, 768, 10)
    onet, pnet = onets.MLP(sizes), be.nn.MLP(sizes)
    P = synth.make_params(onet.param_specs(), 34)
    pnet.load(P)
    x = be.tensor(synth.bf16_values(synth.normal((128, 512), 34, 1)), dtype="bf16")
    y = be.tensor(synth.labels(128, 10, 34))
    params = pnet.parameters()
    if overlap:
        be.sgd_overlap(params, LR, MU, WD)
    bufs = None
    try:
        for step in range(3):
            before = {k: p.numpy().astype(np.float64) for k, p in pnet.params.items()}
            vbefore = {k: be.sgd_momentum(p) for k, p in pnet.params.items()}
            vbefore = {k: v.numpy().astype(np.float64) for k, v in vbefore.items() if v is not None}
            be.zero_grad(params)
            loss = pnet.loss(x, y)
            loss.backward()
            if not overlap:
                be.sgd_step(params, LR, MU, WD)
            checked = 0
            for k, p in pnet.params.items():
                if p.grad is None:
                    assert overlap and k.endswith(".w"), k  # fused epilogue: gradient never stored
                    continue
                g = {k: p.grad.numpy().astype(np.float64)}
                newp, newb = oracle_sgd({k: before[k]}, g, LR, MU, WD, {k: vbefore[k]} if k in vbefore else None)
                assert rel(p.numpy(), newp[k]) < 1e-6, (step, k)
                assert rel(be.sgd_momentum(p).numpy(), newb[k]) < 1e-6, (step, "v", k)
                checked += 1
            assert checked >= 3
    finally:
        be.sgd_overlap([])


@pytest.mark.parametrize("shape", [(1024, 4096, 4096), (256, 1024, 512)])
def test_fused_sgd_epilogue_exact_gradient(shape):
    """The wgrad GEMM with the SGD update in its epilogue (C2 4096×4096 and a
    smaller shape; μ=0.9, wd=1e-4, 3 steps).  x and the upstream gradient are
    small integers, so dW = xᵀ·dY is an exact integer in fp32 whatever the
    summation order: the device's fused update is compared with the oracle's
    SGD on that exact gradient (params and momentum at 1e-6), and the bf16
    shadow the next forward reads must be exactly RN-even(master): a forward
    with x = identity rows returns the shadow rows themselves."""
    be = be_init()
    be.set_compute_dtype("bf16")
    B, K, N = shape
    rng = np.random.default_rng(B + K + N)
    xv = rng.integers(-1, 2, (B, K)).astype(np.float32)
    gv = rng.integers(-1, 2, (B, N)).astype(np.float32)
    W0 = synth.normal((K, N), 35, 1000) / np.sqrt(K)
    b0 = synth.normal((N,), 35, 1001) / np.sqrt(K)
    lr = 1e-4
    W = be.tensor(W0, requires_grad=True)
    b = be.tensor(b0, requires_grad=True)
    x = be.tensor(xv, dtype="bf16")
    g = be.tensor(gv, dtype="bf16")
    gW = xv.astype(np.float64).T @ gv.astype(np.float64)     # exact
    gb = gv.astype(np.float64).sum(0)
    be.sgd_overlap([W, b], lr, MU, WD)
    op = {"W": W0.astype(np.float64), "b": b0.astype(np.float64)}
    bufs = None
    try:
        for step in range(3):
            y = be.linear(x, W, b)
            y.backward(g)
            op, bufs = oracle_sgd(op, {"W": gW, "b": gb}, lr, MU, WD, bufs)
            assert W.grad is None, "the weight update must run in the wgrad epilogue"
            assert rel(W.numpy(), op["W"]) < 1e-6, step
            assert rel(be.sgd_momentum(W).numpy(), bufs["W"]) < 1e-6, step
            assert rel(b.numpy(), op["b"]) < 1e-6, step
            be.zero_grad([b])
    finally:
        be.sgd_overlap([])
    # shadow check: rows of the identity select rows of the bf16 shadow exactly
    rows = min(K, 256)
    eye = np.zeros((rows, K), np.float32)
    eye[np.arange(rows), np.arange(rows)] = 1.0
    with be.no_grad():
        ysel = be.linear(be.tensor(eye, dtype="bf16"), W, None).numpy()
    assert np.array_equal(ysel, synth.bf16_values(W.numpy()[:rows]))
