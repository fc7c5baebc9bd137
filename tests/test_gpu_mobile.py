"""Parity of the Table 1 CNN extras on the B200 (-m gpu): inverted dropout
with its counter-based mask (bit-exact keep decisions), the depthwise
convolution (forward, dgrad, wgrad), batch norm with fused ReLU6, and whole
training steps of small VGG-19 / MobileNetV2 nets, against the float64
oracle (oracle/ops.py dropout, conv2d_depthwise, relu6; oracle/nets.py)."""
import numpy as np
import pytest

import synth
from gpu_common import be_init, rel, run_product_step, compare_step
from oracle import ops as oops, nets as onets
from oracle.autograd import Var, backward
from oracle.step import train_step

pytestmark = pytest.mark.gpu

TOL = {"bf16": 2e-2, "f32": 1e-4}


def nchw_to_nhwc(a):
    return np.ascontiguousarray(np.asarray(a).transpose(0, 2, 3, 1))


def nhwc_to_nchw(a):
    return np.ascontiguousarray(np.asarray(a).transpose(0, 3, 1, 2))


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("shape,p,seed,offset", [((256, 4096), 0.5, 3, 6), ((37, 1280), 0.2, 11, 0),
                                                 ((1, 3), 0.9, 7, 1), ((5, 7, 3), 0.5, 2**40 + 5, 2**33),
                                                 ((0, 8), 0.5, 1, 0)])
def test_dropout_mask_bit_exact_and_grads(shape, p, seed, offset, dtype):
    """Forward values, keep decisions (bit-exact, every element), and the
    regenerated mask in backward: dx = dy·keep/(1−p)."""
    be = be_init()
    n = int(np.prod(shape))
    x = synth.normal(shape, 41, 1) + 3.0  # nonzero everywhere: y ≠ 0 ⇔ kept
    if dtype == "bf16":
        x = synth.bf16_values(x)
    xl = be.tensor(x, requires_grad=True)
    xd = be.cast(xl, "bf16") if dtype == "bf16" else xl
    y = be.dropout(xd, p, seed, offset)
    yd = y.numpy()
    keep = oops.dropout_keep_mask(n, p, seed, offset).reshape(shape)
    assert np.array_equal(yd != 0, keep)
    xo = Var(x.astype(np.float64), True)
    yo = oops.dropout(xo, p, seed, offset)
    assert rel(yd, yo.value) <= (2 ** -8 if dtype == "bf16" else 1e-6)
    if n == 0:
        return
    g = synth.normal(shape, 42, 1)
    if dtype == "bf16":
        g = synth.bf16_values(g)
    y.backward(be.tensor(g, dtype="bf16" if dtype == "bf16" else None))
    backward(yo, g.astype(np.float64))
    assert rel(xl.grad.numpy(), xo.grad) <= (2 ** -8 if dtype == "bf16" else 1e-6)
    assert np.array_equal(xl.grad.numpy() != 0, keep)


def test_dropout_eval_and_p0_are_identity():
    """training=False and p = 0 return x bitwise."""
    be = be_init()
    x = synth.normal((9, 33), 43, 1)
    for kw in (dict(p=0.5, training=False), dict(p=0.0, training=True)):
        y = be.dropout(be.tensor(x), kw["p"], 5, 0, kw["training"]).numpy()
        assert np.array_equal(y, x)
    assert not be.dropout(be.tensor(x), 1.0, 5, 0).numpy().any()


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("geom", [(2, 16, 9, 9, 1), (2, 24, 10, 10, 2), (3, 144, 7, 7, 2), (1, 960, 7, 7, 1),
                                  (2, 8, 5, 6, 1), (1, 40, 11, 13, 2), (4, 32, 1, 1, 1)])
def test_depthwise_conv_op(geom, dtype):
    """Depthwise 3×3 (pad 1) forward, dx, dw vs the oracle (several channel
    groups, ragged spatial sizes, stride 1 and 2, a 1×1 map)."""
    be = be_init()
    be.set_compute_dtype(dtype)
    N, C, H, W, st = geom
    x = synth.normal((N, C, H, W), 44, 1)
    w = synth.normal((C, 1, 3, 3), 44, 2) / 3.0
    if dtype == "bf16":
        x = synth.bf16_values(x)
    xl = be.tensor(nchw_to_nhwc(x), requires_grad=True)
    xd = be.cast(xl, "bf16") if dtype == "bf16" else xl
    wd = be.tensor(np.ascontiguousarray(w[:, 0].transpose(1, 2, 0)), requires_grad=True)
    y = be.conv2d_depthwise(xd, wd, st, 1)
    xo, wo = Var(x.astype(np.float64), True), Var(w.astype(np.float64), True)
    yo = oops.conv2d_depthwise(xo, wo, st, 1)
    tol = TOL[dtype]
    assert rel(nhwc_to_nchw(y.numpy()), yo.value) <= tol
    g = synth.normal(yo.value.shape, 44, 3)
    if dtype == "bf16":
        g = synth.bf16_values(g)
    y.backward(be.tensor(nchw_to_nhwc(g), dtype="bf16" if dtype == "bf16" else None))
    backward(yo, g.astype(np.float64))
    assert rel(nhwc_to_nchw(xl.grad.numpy()), xo.grad) <= tol
    assert rel(wd.grad.numpy(), wo.grad[:, 0].transpose(1, 2, 0)) <= tol


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("st", [1, 2])
@pytest.mark.parametrize("geom", [(2, 24, 10, 10), (1, 40, 11, 13), (2, 96, 1, 3), (3, 16, 7, 2), (1, 32, 17, 5)])
def test_depthwise_dgrad_accumulates(geom, st, dtype):
    """dx (stride 2: the 2×2-quad kernel; stride 1: the column-strip kernel)
    written fresh by the first VJP and accumulated (beta 1) by the second: x
    feeds two depthwise convs with different filters; ragged odd / tiny maps,
    maps taller than one strip; dw of both filters."""
    be = be_init()
    be.set_compute_dtype(dtype)
    N, C, H, W = geom
    x = synth.normal((N, C, H, W), 46, 1)
    w1 = synth.normal((C, 1, 3, 3), 46, 2) / 3.0
    w2 = synth.normal((C, 1, 3, 3), 46, 3) / 3.0
    if dtype == "bf16":
        x = synth.bf16_values(x)
    xl = be.tensor(nchw_to_nhwc(x), requires_grad=True)
    xd = be.cast(xl, "bf16") if dtype == "bf16" else xl
    wl = [be.tensor(np.ascontiguousarray(w[:, 0].transpose(1, 2, 0)), requires_grad=True) for w in (w1, w2)]
    y = be.add(be.conv2d_depthwise(xd, wl[0], st, 1), be.conv2d_depthwise(xd, wl[1], st, 1))
    xo = Var(x.astype(np.float64), True)
    wo = [Var(w.astype(np.float64), True) for w in (w1, w2)]
    yo = oops.add(oops.conv2d_depthwise(xo, wo[0], st, 1), oops.conv2d_depthwise(xo, wo[1], st, 1))
    g = synth.normal(yo.value.shape, 46, 4)
    if dtype == "bf16":
        g = synth.bf16_values(g)
    y.backward(be.tensor(nchw_to_nhwc(g), dtype="bf16" if dtype == "bf16" else None))
    backward(yo, g.astype(np.float64))
    assert rel(nhwc_to_nchw(xl.grad.numpy()), xo.grad) <= TOL[dtype]
    for a, b in zip(wl, wo):
        assert rel(a.grad.numpy(), b.grad[:, 0].transpose(1, 2, 0)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("C", [32, 96, 144])
def test_batchnorm_relu6(C, dtype):
    """BN with the fused ReLU6 (act = 2): forward clamp and the backward mask
    0 < y < 6 (recomputed in the BN backward passes), vs oracle BN + relu6."""
    be = be_init()
    be.set_compute_dtype(dtype)
    N, H, W = 4, 6, 5
    x = synth.normal((N, C, H, W), 45, 1) * 4.0 + 1.0  # plenty of values above 6 and below 0
    if dtype == "bf16":
        x = synth.bf16_values(x)
    gam = (synth.normal((C,), 45, 2) * 2.0 + 3.0).astype(np.float32)
    bet = synth.normal((C,), 45, 3)
    xl = be.tensor(nchw_to_nhwc(x), requires_grad=True)
    xd = be.cast(xl, "bf16") if dtype == "bf16" else xl
    gl, bl = be.tensor(gam, requires_grad=True), be.tensor(bet, requires_grad=True)
    y = be.batchnorm2d(xd, gl, bl, act=2)
    yd = nhwc_to_nchw(y.numpy())
    xo, go, bo = (Var(a.astype(np.float64), True) for a in (x, gam, bet))
    zo, _ = oops.batchnorm2d(xo, go, bo)
    yo = oops.relu6(zo)
    tol = TOL[dtype]
    assert rel(yd, yo.value) <= tol
    assert yd.max() <= 6.0 and yd.min() >= 0.0 and (yd == 6.0).any()
    g = synth.normal(yd.shape, 45, 4)
    if dtype == "bf16":
        g = synth.bf16_values(g)
    y.backward(be.tensor(nchw_to_nhwc(g), dtype="bf16" if dtype == "bf16" else None))
    # the mask the device used is decided from its own output (SURVEY §8(c) reading 16)
    zo2, _ = oops.batchnorm2d(xo2 := Var(x.astype(np.float64), True), go2 := Var(gam.astype(np.float64), True),
                              bo2 := Var(bet.astype(np.float64), True))
    backward(zo2, g.astype(np.float64) * ((yd > 0) & (yd < 6)))
    assert rel(nhwc_to_nchw(xl.grad.numpy()), xo2.grad) <= tol
    assert rel(gl.grad.numpy(), go2.grad) <= tol
    assert rel(bl.grad.numpy(), bo2.grad) <= tol


def _small_mobilenet(be):
    settings = ((1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 2, 2))
    return (onets.MobileNetV2(classes=10, width=0.5, settings=settings, dropout=0.2, seed=9),
            be.nn.MobileNetV2(classes=10, width=0.5, settings=settings, dropout=0.2, seed=9))


def _small_vgg(be):
    return (onets.VGG19(classes=10, width=1 / 8, image=32, dropout=0.5, seed=4),
            be.nn.VGG19(classes=10, width=1 / 8, image=32, dropout=0.5, seed=4))


def test_small_vgg_one_step_fp32():
    """One fp32 (3xTF32) SGD step of a reduced VGG-19 (dropout on, the same
    counter-based masks on both sides) vs the oracle at 1e-4, every tensor."""
    be = be_init()
    be.set_compute_dtype("f32")
    onet, pnet = _small_vgg(be)
    x, y = synth.normal((4, 3, 32, 32), 46, 1), synth.labels(4, 10, 46)
    P = synth.make_params(onet.param_specs(), 46)
    ref = train_step(onet, P, (x, y), lr=0.01)
    loss, grads, new = run_product_step(be, pnet, P, (be.nn.images_to_device(x, "f32"), be.tensor(y)))
    compare_step(ref, loss, grads, new, 1e-4)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_small_mobilenet_one_step(dtype):
    """One SGD step of a reduced MobileNetV2 (batch 8, 32²): the loss and every
    tensor whose conditioning floor allows it (tests/conditioning.py) at the
    north_star tolerance; the BN-β gradients behind a linear conv → BN path
    are exactly 0 in exact arithmetic (Σ dy over a normalised channel), so
    they are gated only through κ (reading R16)."""
    from gpu_common import e2e_gate
    be = be_init()
    be.set_compute_dtype(dtype)
    onet, pnet = _small_mobilenet(be)
    x, y = synth.normal((8, 3, 32, 32), 47, 1), synth.labels(8, 10, 47)
    if dtype == "bf16":
        x = synth.bf16_values(x)
    P = synth.make_params(onet.param_specs(), 47)
    e2e_gate(be, onet, pnet, P, (x, y), (be.nn.images_to_device(x, dtype), be.tensor(y)), dtype, name="mobilenet")
