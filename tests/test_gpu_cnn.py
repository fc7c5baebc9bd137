"""CNN / recommender parity on the B200 (-m gpu): conv2d (fwd, dgrad, wgrad),
max / average pooling, batch norm, residual add, embedding — per op and
whole training steps — against the float64 oracle.  Index tensors (im2col
offsets, max-pool argmax) must match bit-exactly."""
import numpy as np
import pytest

import synth
from gpu_common import be_init, rel, run_product_step, compare_step
from oracle import ops as oops, nets as onets
from oracle.autograd import Var, backward
from oracle.step import train_step

pytestmark = pytest.mark.gpu


def nchw_to_nhwc(a):
    return np.ascontiguousarray(np.asarray(a).transpose(0, 2, 3, 1))


def nhwc_to_nchw(a):
    return np.ascontiguousarray(np.asarray(a).transpose(0, 3, 1, 2))


@pytest.mark.parametrize("geom", [(2, 3, 5, 5, 3, 3, 1, 1), (2, 8, 9, 7, 3, 3, 2, 1), (1, 4, 11, 11, 11, 11, 4, 2),
                                  (3, 16, 6, 6, 1, 1, 2, 0), (1, 1, 28, 28, 3, 3, 1, 0)])
def test_im2col_offsets_bit_exact(geom):
    be = be_init()
    N, C, H, W, R, S, st, pd = geom
    dev = be.im2col_offsets(N, C, H, W, R, S, st, pd)
    ref = oops.im2col_table(N, C, H, W, R, S, st, pd)
    assert np.array_equal(dev, ref)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("geom", [
    (2, 64, 9, 9, 64, 3, 1, 1),      # bf16: shared-patch stride-1 kernel (C = K = 64)
    (2, 64, 10, 10, 128, 3, 2, 1),   # TMA-im2col implicit GEMM (C % 64 == 0), stride 2
    (1, 128, 7, 7, 128, 3, 1, 1),    # TMA-im2col, C = K = 128
    (2, 8, 40, 40, 64, 7, 2, 3),     # stem (C = 8, K = 64, stride 2): phase-split patch
    (1, 8, 35, 35, 64, 11, 4, 2),    # AlexNet-conv1-like (small-C gather)
    (1, 16, 9, 11, 48, 3, 1, 1),     # small-C gather, stride 1
    (2, 256, 6, 6, 64, 1, 2, 0)])    # 1×1 stride 2
def test_conv_kernels_gather_offsets_bit_exact(geom, dtype):
    """Index parity of the conv kernels themselves (not a side kernel): with
    one-hot weights (output channel k selects column j0 + k of the im2col
    matrix) and an input holding base-b digits of (NHWC offset + 1), every
    output element is exactly one gathered input value; the digits
    reassemble the offset table the kernel used, which must equal the
    oracle's im2col_table bit-exactly (−1 in the padding).  b = 128 in bf16
    (integers ≤ 256 are exact), 2048 with 3xTF32."""
    be = be_init()
    be.set_compute_dtype(dtype)
    N, C, H, W, K, R, st, pd = geom
    P, Q = (H + 2 * pd - R) // st + 1, (W + 2 * pd - R) // st + 1
    RSC = R * R * C
    base = 128 if dtype == "bf16" else 2048
    off1 = np.arange(1, N * H * W * C + 1, dtype=np.int64).reshape(N, H, W, C)  # NHWC offset + 1
    nd = 1
    while base ** nd <= off1.max():
        nd += 1
    digits = [((off1 // base ** d) % base).astype(np.float32) for d in range(nd)]
    xs = [be.tensor(dg, dtype=dtype) for dg in digits]
    got = np.zeros((N * P * Q, RSC), np.int64)
    for j0 in range(0, RSC, K):
        wk = np.zeros((K, RSC), np.float32)
        cols = np.arange(j0, min(j0 + K, RSC))
        wk[cols - j0, cols] = 1.0
        wd = be.tensor(wk.reshape(K, R, R, C))          # KRSC
        acc = np.zeros((N * P * Q, K), np.int64)
        for d, x in enumerate(xs):
            y = be.conv2d(x, wd, None, st, pd).numpy().reshape(N * P * Q, K)
            assert np.array_equal(y, np.round(y))
            acc += y.astype(np.int64) * base ** d
        got[:, cols] = acc[:, :len(cols)]
    ref = oops.im2col_table(N, C, H, W, R, R, st, pd)
    assert np.array_equal(got - 1, ref)


@pytest.mark.parametrize("cfg", [(2, 8, 9, 9, 16, 3, 1, 1), (2, 8, 10, 10, 12, 3, 2, 1), (3, 16, 7, 7, 32, 1, 1, 0),
                                 (2, 16, 8, 8, 24, 1, 2, 0), (2, 8, 23, 23, 16, 11, 4, 2), (1, 8, 12, 12, 8, 5, 1, 2)])
@pytest.mark.parametrize("act", [0, 1])
def test_conv_op_fp32(cfg, act):
    """conv2d forward + backward (dX, dW, db) in f32 (3xTF32) at 1e-4."""
    be = be_init()
    be.set_compute_dtype("f32")
    N, C, H, W, K, R, st, pd = cfg
    rng = np.random.default_rng(sum(cfg) + act)
    x = rng.standard_normal((N, C, H, W)).astype(np.float32)
    w = (rng.standard_normal((K, C, R, R)) / np.sqrt(C * R * R)).astype(np.float32)
    b = rng.standard_normal(K).astype(np.float32)
    xo, wo, bo = Var(x.astype(np.float64), True), Var(w.astype(np.float64), True), Var(b.astype(np.float64), True)
    yo = oops.conv2d(xo, wo, bo, st, pd)
    if act:
        yo = oops.relu(yo)
    g = rng.standard_normal(yo.value.shape)
    backward(yo, g)
    xd = be.tensor(nchw_to_nhwc(x), requires_grad=True)
    wd = be.tensor(nchw_to_nhwc(w), requires_grad=True)
    bd = be.tensor(b, requires_grad=True)
    yd = be.conv2d(xd, wd, bd, st, pd, act=act)
    yd.backward(be.tensor(nchw_to_nhwc(g).astype(np.float32)))
    assert rel(nhwc_to_nchw(yd.numpy()), yo.value) < 1e-4
    assert rel(nhwc_to_nchw(xd.grad.numpy()), xo.grad) < 1e-4
    assert rel(nhwc_to_nchw(wd.grad.numpy()), wo.grad) < 1e-4
    assert rel(bd.grad.numpy(), bo.grad) < 1e-4


@pytest.mark.parametrize("cfg", [(2, 64, 9, 9, 64, 3, 1, 1), (2, 64, 10, 10, 128, 3, 2, 1), (1, 128, 7, 7, 256, 3, 1, 1),
                                 (2, 64, 14, 14, 64, 1, 2, 0), (3, 64, 17, 13, 96, 3, 1, 1), (1, 192, 5, 5, 320, 3, 1, 1),
                                 # small-C gather kernel (channel-padded conv1: ResNet 7×7/2, AlexNet 11×11/4)
                                 (3, 8, 40, 40, 64, 7, 2, 3), (2, 8, 35, 35, 64, 11, 4, 2), (1, 16, 9, 11, 48, 3, 1, 1),
                                 # phase-split patch kernel (C = 8, K = 64, stride > 1): ResNet conv1 at full
                                 # width (Q = 112), Q = 125 (MMA rows 125..127 discarded), stride 3, AlexNet conv1
                                 (2, 8, 224, 224, 64, 7, 2, 3), (1, 8, 250, 250, 64, 7, 2, 3), (2, 8, 20, 23, 64, 5, 3, 1),
                                 (1, 8, 224, 224, 64, 11, 4, 2),
                                 # shared-patch stride-1 kernel (C = K = 64): ResNet layer-1 size, ragged row groups
                                 (2, 64, 56, 56, 64, 3, 1, 1), (1, 64, 30, 20, 64, 3, 1, 1), (2, 64, 12, 12, 64, 2, 1, 0),
                                 (2, 32, 8, 8, 160, 3, 2, 1), (1, 8, 6, 6, 16, 5, 1, 0),
                                 # TMA-im2col kernel at ResNet layer-2/3/4 and VGG shapes (C ≥ 128), ragged
                                 # rows and columns, K = 512 (two N tiles), 1×1 and 2×2 filters
                                 (2, 128, 28, 28, 128, 3, 1, 1), (2, 256, 14, 14, 256, 3, 1, 1),
                                 (1, 512, 7, 7, 512, 3, 1, 1), (1, 128, 60, 50, 128, 3, 1, 1),
                                 (1, 128, 13, 11, 256, 3, 1, 1), (2, 256, 20, 9, 128, 3, 1, 1),
                                 (1, 192, 17, 30, 128, 2, 1, 0), (3, 128, 9, 9, 256, 1, 1, 0)])
def test_conv_op_bf16_implicit_gemm(cfg):
    """bf16 conv forward through the implicit-GEMM kernel (cp.async gather, no
    im2col) vs the oracle on the same bf16-rounded x and W: fp32 accumulate,
    one bf16 rounding of the output (≤ 2^-8 relative) → gate 1e-2."""
    be = be_init()
    be.set_compute_dtype("bf16")
    N, C, H, W, K, R, st, pd = cfg
    rng = np.random.default_rng(sum(cfg))
    from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
    q = lambda a: bf16_bits_to_f32(f32_to_bf16_bits(a.astype(np.float32)))
    x = q(rng.standard_normal((N, C, H, W)))
    w = q(rng.standard_normal((K, C, R, R)) / np.sqrt(C * R * R))
    b = rng.standard_normal(K).astype(np.float32)
    xo, wo = Var(x.astype(np.float64), True), Var(w.astype(np.float64), True)
    yo = oops.conv2d(xo, wo, Var(b.astype(np.float64)), st, pd)
    calls0 = be.launch_count()
    xd = be.tensor(nchw_to_nhwc(x), requires_grad=True)
    wd = be.tensor(nchw_to_nhwc(w), requires_grad=True)
    yd = be.conv2d(be.cast(xd, "bf16"), wd, be.tensor(b), st, pd, act=0)
    assert rel(nhwc_to_nchw(yd.numpy()), yo.value) < 1e-2
    assert be.launch_count() - calls0 <= 4  # input cast, weight shadow cast, one conv kernel (no im2col)
    # backward with a bf16 upstream: dgrad (stride 1 → flipped-weight implicit conv) and wgrad
    g = q(rng.standard_normal(yo.value.shape))
    backward(yo, g.astype(np.float64))
    yd.backward(be.tensor(nchw_to_nhwc(g), dtype="bf16"))
    assert rel(nhwc_to_nchw(xd.grad.numpy()), xo.grad) < 1e-2
    assert rel(nhwc_to_nchw(wd.grad.numpy()), wo.grad) < 1e-3


@pytest.mark.parametrize("R,pd", [(1, 0), (3, 1)])
@pytest.mark.parametrize("H", [14, 15])
def test_conv_stride2_dgrad_accumulates(R, pd, H):
    """Stride-2 dgrad through dcols + the stride-2 col2im kernel, accumulated
    into a gradient another consumer already wrote (x feeds a 1×1 stride-1
    conv and the stride-2 conv, as a ResNet block input feeds conv1 and the
    down-sampling shortcut): pixels no stride-2 tap reaches keep the first
    consumer's gradient.  Odd H: the last row / column has no tap for R = 1."""
    be = be_init()
    be.set_compute_dtype("bf16")
    from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
    q = lambda a: bf16_bits_to_f32(f32_to_bf16_bits(a.astype(np.float32)))
    rng = np.random.default_rng(R * 100 + H)
    N, C, K = 2, 64, 128
    x = q(rng.standard_normal((N, C, H, H)))
    w1 = q(rng.standard_normal((64, C, 1, 1)) / np.sqrt(C))
    w2 = q(rng.standard_normal((K, C, R, R)) / np.sqrt(C * R * R))
    xo = Var(x.astype(np.float64), True)
    y1 = oops.conv2d(xo, Var(w1.astype(np.float64)), None, 1, 0)
    y2 = oops.conv2d(xo, Var(w2.astype(np.float64)), None, 2, pd)
    g1 = q(rng.standard_normal(y1.value.shape))
    g2 = q(rng.standard_normal(y2.value.shape))
    backward(y1, g1.astype(np.float64))
    backward(y2, g2.astype(np.float64))
    xd = be.tensor(nchw_to_nhwc(x), requires_grad=True)
    xb = be.cast(xd, "bf16")
    z1 = be.conv2d(xb, be.tensor(nchw_to_nhwc(w1)), None, 1, 0)
    z2 = be.conv2d(xb, be.tensor(nchw_to_nhwc(w2)), None, 2, pd)
    loss = be.add(be.sum(be.mul(z1, be.tensor(nchw_to_nhwc(g1), dtype="bf16"))),
                  be.sum(be.mul(z2, be.tensor(nchw_to_nhwc(g2), dtype="bf16"))))
    loss.backward()
    assert rel(nhwc_to_nchw(xd.grad.numpy()), xo.grad) < 1e-2


@pytest.mark.parametrize("cfg", [
    # (N, C, H, W, K, R, stride, pad): ResNet-50 v1.5 stride-2 3×3 (layers 2-4) and 1×1 projections
    (2, 128, 56, 56, 128, 3, 2, 1), (2, 256, 28, 28, 256, 3, 2, 1), (4, 512, 14, 14, 512, 3, 2, 1),
    (2, 256, 56, 56, 512, 1, 2, 0), (2, 1024, 14, 14, 2048, 1, 2, 0),
    # odd sizes (phases of unequal height), pad 0 and 2, 5×5, stride 3 (nine phases, some empty)
    (1, 96, 15, 13, 64, 3, 2, 1), (2, 64, 17, 17, 128, 3, 2, 0), (1, 48, 19, 16, 192, 5, 2, 2),
    (1, 64, 20, 22, 64, 3, 3, 1), (2, 32, 9, 9, 64, 2, 3, 0)])
@pytest.mark.parametrize("first", [True, False])
def test_conv_dgrad_phases(cfg, first):
    """Stride ≥ 2 data gradient as stride² phase convolutions (conv_dgrad_phases):
    every phase's implicit GEMM stores its rows straight into dx.  `first`:
    the stride-2 conv's backward runs first (beta 0: phases without taps are
    zero-filled) or after a 1×1 consumer of the same input (beta 1: its live
    phases accumulate, the rest keep the other consumer's gradient).  Against
    the float64 oracle on the same bf16 inputs: fp32 accumulate, one bf16
    rounding of each stored gradient (≤ 2^-8 relative) → 1e-2."""
    be = be_init()
    be.set_compute_dtype("bf16")
    from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
    q = lambda a: bf16_bits_to_f32(f32_to_bf16_bits(a.astype(np.float32)))
    N, C, H, W, K, R, st, pd = cfg
    rng = np.random.default_rng(sum(cfg) + first)
    x = q(rng.standard_normal((N, C, H, W)))
    w1 = q(rng.standard_normal((64, C, 1, 1)) / np.sqrt(C))
    w2 = q(rng.standard_normal((K, C, R, R)) / np.sqrt(C * R * R))
    xo = Var(x.astype(np.float64), True)
    y1 = oops.conv2d(xo, Var(w1.astype(np.float64)), None, 1, 0)
    y2 = oops.conv2d(xo, Var(w2.astype(np.float64)), None, st, pd)
    g1 = q(rng.standard_normal(y1.value.shape))
    g2 = q(rng.standard_normal(y2.value.shape))
    backward(y1, g1.astype(np.float64))
    backward(y2, g2.astype(np.float64))
    xd = be.tensor(nchw_to_nhwc(x), requires_grad=True)
    xb = be.cast(xd, "bf16")
    # the engine runs the later-recorded consumer's backward first
    if first:
        z1 = be.conv2d(xb, be.tensor(nchw_to_nhwc(w1)), None, 1, 0)
        z2 = be.conv2d(xb, be.tensor(nchw_to_nhwc(w2)), None, st, pd)
    else:
        z2 = be.conv2d(xb, be.tensor(nchw_to_nhwc(w2)), None, st, pd)
        z1 = be.conv2d(xb, be.tensor(nchw_to_nhwc(w1)), None, 1, 0)
    l1 = be.sum(be.mul(z1, be.tensor(nchw_to_nhwc(g1), dtype="bf16")))
    l2 = be.sum(be.mul(z2, be.tensor(nchw_to_nhwc(g2), dtype="bf16")))
    loss = be.add(l1, l2) if first else be.add(l2, l1)
    loss.backward()
    assert rel(nhwc_to_nchw(xd.grad.numpy()), xo.grad) < 1e-2


@pytest.mark.parametrize("C", [5, 16])
@pytest.mark.parametrize("k,s,p", [(3, 2, 0), (3, 2, 1)])
def test_maxpool_op_and_argmax_bit_exact(k, s, p, C):
    be = be_init()
    be.set_compute_dtype("f32")
    rng = np.random.default_rng(k + s + p)
    x = rng.standard_normal((2, C, 13, 13)).astype(np.float32)
    x[0, 0, :4, :4] = 0.0  # tied windows → first index
    xo = Var(x.astype(np.float64), True)
    yo, am = oops.maxpool2d(xo, k, s, p)
    g = rng.standard_normal(yo.value.shape)
    backward(yo, g)
    xd = be.tensor(nchw_to_nhwc(x), requires_grad=True)
    yd, amd = be.maxpool2d(xd, k, s, p, with_argmax=True)
    yd.backward(be.tensor(nchw_to_nhwc(g).astype(np.float32)))
    assert np.array_equal(nhwc_to_nchw(yd.numpy()), yo.value.astype(np.float32))
    # device window index (r*k+u) → plane index h*W+w, compared bit-exactly
    win = nhwc_to_nchw(amd.numpy()).astype(np.int64)
    P = yo.value.shape[2]
    pi = np.arange(P)[:, None]
    qi = np.arange(P)[None, :]
    h = pi * s - p + win // k
    w = qi * s - p + win % k
    assert np.array_equal(h * x.shape[3] + w, am)
    assert rel(nhwc_to_nchw(xd.grad.numpy()), xo.grad) < 1e-6


@pytest.mark.parametrize("C,H", [(16, 13), (64, 14), (8, 57)])
@pytest.mark.parametrize("k,s,p", [(3, 2, 0), (3, 2, 1), (2, 2, 0)])
def test_maxpool_bf16_rows_bit_exact(k, s, p, C, H):
    """bf16 max pool (the row kernels maxpool_fwd_rows / maxpool_bwd_rows):
    pooled values and winners bit-exact against the oracle on the same
    bf16-valued input (ties → first index); dx = Σ of the winners' upstream
    (≤ 4 bf16 terms, fp32 sum, one rounding) within one bf16 ulp."""
    from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
    be = be_init()
    be.set_compute_dtype("bf16")
    q = lambda a: bf16_bits_to_f32(f32_to_bf16_bits(np.asarray(a, np.float32)))
    rng = np.random.default_rng(C + H + k + s + p)
    x = q(rng.standard_normal((3, C, H, H)))
    x[0, :, :5, :5] = 0.5  # tied windows → first index
    xo = Var(x.astype(np.float64), True)
    yo, am = oops.maxpool2d(xo, k, s, p)
    g = q(rng.standard_normal(yo.value.shape))
    backward(yo, g.astype(np.float64))
    xd = be.tensor(nchw_to_nhwc(x), requires_grad=True)
    yd, amd = be.maxpool2d(be.cast(xd, "bf16"), k, s, p, with_argmax=True)
    yd.backward(be.tensor(nchw_to_nhwc(g), dtype="bf16"))
    assert np.array_equal(nhwc_to_nchw(yd.numpy()).astype(np.float64), yo.value)
    win = nhwc_to_nchw(amd.numpy()).astype(np.int64)
    P = yo.value.shape[2]
    hh = np.arange(P)[:, None] * s - p + win // k
    ww = np.arange(P)[None, :] * s - p + win % k
    assert np.array_equal(hh * H + ww, am)
    assert rel(nhwc_to_nchw(xd.grad.numpy()), xo.grad) < 8e-3


@pytest.mark.parametrize("C", [6, 24])
def test_avgpool_bn_add_ops_fp32(C):
    be = be_init()
    be.set_compute_dtype("f32")
    rng = np.random.default_rng(11)
    x = (rng.standard_normal((4, C, 5, 5)) * 2 + 0.5).astype(np.float32)
    r = rng.standard_normal((4, C, 5, 5)).astype(np.float32)
    gam = (rng.standard_normal(C) + 1).astype(np.float32)
    bet = rng.standard_normal(C).astype(np.float32)
    xo, ro = Var(x.astype(np.float64), True), Var(r.astype(np.float64), True)
    go, bo = Var(gam.astype(np.float64), True), Var(bet.astype(np.float64), True)
    yo, (rm, rv) = oops.batchnorm2d(xo, go, bo)
    zo = oops.avgpool_global(oops.relu(oops.add(yo, ro)))
    g = rng.standard_normal(zo.value.shape)
    backward(zo, g)
    xd, rd = be.tensor(nchw_to_nhwc(x), requires_grad=True), be.tensor(nchw_to_nhwc(r), requires_grad=True)
    gd, bd = be.tensor(gam, requires_grad=True), be.tensor(bet, requires_grad=True)
    rmd, rvd = be.tensor(np.zeros(C, np.float32)), be.tensor(np.ones(C, np.float32))
    yd = be.batchnorm2d(xd, gd, bd, rmd, rvd)
    zd = be.avgpool_global(be.add_relu(yd, rd))
    zd.backward(be.tensor(g.astype(np.float32)))
    assert rel(zd.numpy(), zo.value) < 1e-5
    for dev, orc in ((xd, xo), (rd, ro), (gd, go), (bd, bo)):
        d = dev.grad.numpy()
        assert rel(nhwc_to_nchw(d) if d.ndim == 4 else d, orc.grad) < 1e-4
    assert rel(rmd.numpy(), rm) < 1e-5 and rel(rvd.numpy(), rv) < 1e-5


def test_embedding_op_deterministic():
    be = be_init()
    be.set_compute_dtype("f32")
    rng = np.random.default_rng(12)
    E = rng.standard_normal((97, 24)).astype(np.float32)
    ids = rng.integers(0, 97, 3000).astype(np.int32)
    ids[:50] = 5  # a hot row
    g = rng.standard_normal((3000, 24))
    Eo = Var(E.astype(np.float64), True)
    backward(oops.embedding(Eo, ids), g)
    grads = []
    for _ in range(2):
        Ed = be.tensor(E, requires_grad=True)
        rows = be.embedding(Ed, be.tensor(ids))
        assert np.array_equal(rows.numpy(), E[ids])
        rows.backward(be.tensor(g.astype(np.float32)))
        grads.append(Ed.grad.numpy())
    assert np.array_equal(grads[0], grads[1])  # bitwise reproducible
    assert rel(grads[0], Eo.grad) < 1e-5


# ------------------------------------------------------------ whole training steps (fp32 at 1e-4)
def _step_case(onet, pnet, batch_o, batch_d, dtype="f32", seed=0, tol=1e-4):
    be = be_init()
    be.set_compute_dtype(dtype)
    assert onet.param_specs() == pnet.param_specs()
    P = synth.make_params(onet.param_specs(), seed)
    ref = train_step(onet, P, batch_o, lr=0.01)
    loss, grads, new = run_product_step(be, pnet, P, batch_d)
    return compare_step(ref, loss, grads, new, tol)


def test_listing1_net_fp32():
    be = be_init()
    x = synth.uniform((8, 1, 28, 28), 0, 1)
    y = synth.labels(8, 10, 0)
    errs = _step_case(onets.ListingNet(), be.nn.ListingNet(), (x, y),
                      (be.nn.images_to_device(x, "f32"), be.tensor(y)))
    print("listing max err", max(errs.values()))


def test_alexnet_small_fp32():
    be = be_init()
    x = synth.normal((2, 3, 127, 127), 1, 1)
    y = synth.labels(2, 10, 1)
    errs = _step_case(onets.AlexNet(classes=10, width=1 / 16, image=127),
                      be.nn.AlexNet(classes=10, width=1 / 16, image=127), (x, y),
                      (be.nn.images_to_device(x, "f32"), be.tensor(y)), seed=1)
    print("alexnet max err", max(errs.values()))


def test_resnet_small_fp32():
    be = be_init()
    x = synth.normal((4, 3, 64, 64), 2, 1)
    y = synth.labels(4, 10, 2)
    errs = _step_case(onets.ResNet50(layers=(1, 1, 1, 1), base=8, classes=10),
                      be.nn.ResNet50(layers=(1, 1, 1, 1), base=8, classes=10), (x, y),
                      (be.nn.images_to_device(x, "f32"), be.tensor(y)), seed=2)
    print("resnet max err", max(errs.values()))


def test_ncf_small_fp32():
    be = be_init()
    users, items, y = synth.ncf_batch(256, 50, 30, 3)
    onet = onets.NCF(n_users=50, n_items=30, gmf=8, mlp=(16, 16, 8))
    pnet = be.nn.NCF(n_users=50, n_items=30, gmf=8, mlp=(16, 16, 8))
    errs = _step_case(onet, pnet, (users, items, y), (be.tensor(users), be.tensor(items), be.tensor(y)), seed=3)
    print("ncf max err", max(errs.values()))


@pytest.mark.parametrize("cfg", [(2, 64, 14, 14, 64, 1, 1, 0),     # 1×1 s1: plain GEMM (1-CTA / pair)
                                 (3, 64, 17, 13, 96, 3, 1, 1),     # implicit conv, ragged M, N < tile
                                 (2, 256, 16, 16, 160, 1, 2, 0),   # 1×1 s2: implicit conv, 2 column tiles
                                 (2, 8, 40, 40, 64, 7, 2, 3),      # conv1 small-C kernel
                                 (2, 512, 32, 32, 256, 1, 1, 0),   # pair-sized GEMM
                                 (2, 64, 14, 14, 256, 1, 1, 0),    # K-light expansion: statistics pass kept
                                 (2, 64, 30, 30, 64, 3, 1, 1),     # shared-patch kernel (C = K = 64), ragged rows
                                 (2, 64, 56, 56, 64, 3, 1, 1),     # ResNet layer-1 3×3 (shared patch)
                                 (2, 128, 28, 28, 128, 3, 1, 1),   # ResNet layer-2 3×3 (TMA im2col)
                                 (1, 8, 224, 224, 64, 7, 2, 3),    # ResNet stem (phase-split patch kernel)
                                 (3, 256, 14, 14, 64, 1, 1, 0)])   # bottleneck c1: 1×1 reduce, ragged M
def test_bn_statistics_from_conv_epilogue(cfg):
    """conv2d(..., bn_stats=True) → batchnorm2d: the BN takes its mean /
    variance from the conv epilogue's per-column partial sums of the stored
    bf16 output (one launch fewer) and must equal the oracle's BN of the
    device's own conv output (1e-2, bf16), forward and backward."""
    be = be_init()
    be.set_compute_dtype("bf16")
    from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
    q = lambda a: bf16_bits_to_f32(f32_to_bf16_bits(np.asarray(a, np.float32)))
    N, C, H, W, K, R, st, pd = cfg
    rng = np.random.default_rng(sum(cfg) + 7)
    x = q(rng.standard_normal((N, C, H, W)))
    w = q(rng.standard_normal((K, C, R, R)) / np.sqrt(C * R * R))
    gam = (rng.standard_normal(K) * 0.3 + 1).astype(np.float32)
    bet = (rng.standard_normal(K) * 0.3).astype(np.float32)
    xd = be.tensor(nchw_to_nhwc(x), dtype="bf16")
    wd = be.tensor(nchw_to_nhwc(w), requires_grad=True)
    gd, bd = be.tensor(gam, requires_grad=True), be.tensor(bet, requires_grad=True)
    y = be.conv2d(xd, wd, None, st, pd, bn_stats=True)
    l0 = be.launch_count()
    z = be.batchnorm2d(y, gd, bd, act=1)
    n_epi = be.launch_count() - l0  # statistics finalize + apply (no reduction pass) — except where R·S·C < K
    yv = nhwc_to_nchw(y.numpy()).astype(np.float64)
    yo, go, bo = Var(yv, True), Var(gam.astype(np.float64), True), Var(bet.astype(np.float64), True)
    zo = oops.relu(oops.batchnorm2d(yo, go, bo)[0])
    assert rel(nhwc_to_nchw(z.numpy()), zo.value) < 1e-2
    g = q(rng.standard_normal(zo.value.shape))
    backward(zo, g.astype(np.float64))
    z.backward(be.tensor(nchw_to_nhwc(g), dtype="bf16"))
    assert rel(gd.grad.numpy(), go.grad) < 1e-2 and rel(bd.grad.numpy(), bo.grad) < 1e-2
    # the same BN without epilogue statistics agrees to bf16 rounding
    y2 = be.conv2d(xd, wd, None, st, pd)
    l0 = be.launch_count()
    z2 = be.batchnorm2d(y2, gd, bd, act=1)
    n_pass = be.launch_count() - l0  # statistics pass (+ finalize unless BE_BN_FOLD=1) + apply
    # the epilogue statistics remove exactly the statistics pass (the conv
    # skips them where R·S·C < K: the epilogue is the bottleneck there)
    assert n_epi == (n_pass - 1 if C * R * R >= K else n_pass), (n_epi, n_pass)
    assert rel(z2.numpy(), z.numpy()) < 1e-2


@pytest.mark.parametrize("cfg", [(2, 64, 9, 9, 64, 3, 1, 1), (2, 64, 10, 10, 128, 3, 2, 1), (1, 128, 7, 7, 256, 3, 1, 1),
                                 (3, 64, 17, 13, 96, 3, 1, 1), (2, 64, 30, 30, 64, 3, 1, 1), (1, 64, 12, 12, 64, 5, 2, 2),
                                 # shared-patch variant (stride 1, C = K = 64): ResNet layer-1 size, a ragged last
                                 # row group (P = 27, G = 4), a 2×2 kernel (even tap count)
                                 (2, 64, 56, 56, 64, 3, 1, 1), (2, 64, 27, 25, 64, 3, 1, 1), (1, 64, 10, 12, 64, 2, 1, 0),
                                 # C = K = 128 (one tap per MMA, 3 tap groups): ResNet layer-2 size, ragged
                                 (2, 128, 28, 28, 128, 3, 1, 1), (1, 128, 13, 11, 128, 3, 1, 1),
                                 # C = 64, K = 192 (AlexNet conv2 5×5: three dY planes, N = 192, 7 tap groups)
                                 (2, 64, 27, 27, 192, 5, 1, 2),
                                 # im2col gathered in smem (K % 128 == 0): stride 2 ragged, BN = 256 (C % 256 == 0),
                                 # three M tiles (K = 384), BN = 128 with a tap boundary inside no tile
                                 (3, 128, 15, 15, 128, 3, 2, 1), (2, 256, 9, 9, 256, 3, 1, 1),
                                 (1, 256, 12, 10, 384, 3, 1, 1), (2, 128, 8, 8, 256, 3, 1, 1)])
def test_conv_wgrad_variants_bf16(cfg):
    """Conv weight gradient through every autotuned variant (the first calls
    of a shape cycle through them: TMA-im2col B, materialised columns,
    shifted 4-D tiles of dY and x, shared patch, im2col gathered in smem) —
    each call's dW vs the oracle on the same bf16 x and dY (fp32 accumulation
    → 1e-3)."""
    be = be_init()
    be.set_compute_dtype("bf16")
    N, C, H, W, K, R, st, pd = cfg
    rng = np.random.default_rng(sum(cfg) + 3)
    from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
    q = lambda a: bf16_bits_to_f32(f32_to_bf16_bits(a.astype(np.float32)))
    x = q(rng.standard_normal((N, C, H, W)))
    w = q(rng.standard_normal((K, C, R, R)) / np.sqrt(C * R * R))
    xo, wo = Var(x.astype(np.float64)), Var(w.astype(np.float64), True)
    yo = oops.conv2d(xo, wo, None, st, pd)
    g = q(rng.standard_normal(yo.value.shape))
    backward(yo, g.astype(np.float64))
    xd = be.tensor(nchw_to_nhwc(x), dtype="bf16")
    gd = be.tensor(nchw_to_nhwc(g), dtype="bf16")
    for _ in range(6):  # ≥ one call of each of the (up to) three variants
        wd = be.tensor(nchw_to_nhwc(w), requires_grad=True)
        yd = be.conv2d(xd, wd, None, st, pd)
        yd.backward(gd)
        assert rel(nhwc_to_nchw(wd.grad.numpy()), wo.grad) < 1e-3


@pytest.mark.parametrize("cfg", [(2, 64, 14, 14, 256, 1), (3, 128, 9, 7, 512, 1), (2, 256, 7, 7, 1024, 1),
                                 (1, 40, 11, 13, 24, 2), (4, 96, 5, 5, 64, 0)])
def test_bn_conv1x1_fused_operand(cfg):
    """BN (train) → ReLU / ReLU6 / none → 1×1 conv with the BN applied inside
    the GEMM's operand load (BE_OP_BN_CONV1X1): output, dx, dγ, dβ, dW and the
    running statistics vs the unfused device ops (batchnorm2d then conv2d, each
    parity-checked elsewhere) and vs the float64 oracle composition, every op
    of it fed the same inputs (teacher-forced replay)."""
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from teacher import Replay, OpTrace
    be = be_init()
    be.set_compute_dtype("bf16")
    N, C, H, W, K, act = cfg
    rng = np.random.default_rng(sum(cfg))
    from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
    q = lambda a: bf16_bits_to_f32(f32_to_bf16_bits(a.astype(np.float32)))  # noqa: E731
    x = q(rng.standard_normal((N, H, W, C)) * 2 + 0.5)
    gam = (rng.standard_normal(C) * 0.5 + 1.5).astype(np.float32)
    bet = (rng.standard_normal(C) * 0.5).astype(np.float32)
    w = (rng.standard_normal((K, 1, 1, C)) / np.sqrt(C)).astype(np.float32)

    class M:  # the traced "model": one op
        pass
    m = M()
    m.params = {"g": be.tensor(gam, requires_grad=True), "b": be.tensor(bet, requires_grad=True),
                "w": be.tensor(w, requires_grad=True)}
    m.buffers = {"rm": be.tensor(np.zeros(C, np.float32)), "rv": be.tensor(np.ones(C, np.float32))}
    tr = OpTrace(be.api, m)
    xb = be.tensor(x, dtype="bf16")
    tr.ids[id(xb)] = ("param", "x")  # checked like a parameter: its gradient dx is compared
    fused = tr._wrap("bn_conv1x1")
    y = fused(xb, m.params["g"], m.params["b"], m.buffers["rm"], m.buffers["rv"], m.params["w"], act=act)
    g = q(rng.standard_normal(tuple(y.shape)))
    rp = Replay(be, tr, 2e-2)
    rp.grads[tr.recs[-1]["out"]] = g.astype(np.float64)
    rp.run()
    bad = rp.failures()
    assert not bad, bad
    got = {w_ for (_, _, w_, _) in rp.errs}
    assert {"y", "dx:x", "dgamma:g", "dbeta:b", "dw:w", "running_mean", "running_var"} <= got, got


@pytest.mark.parametrize("cfg", [(2, 256, 14, 14, 256, 3, 1, 1), (1, 512, 7, 9, 512, 3, 1, 1), (2, 192, 15, 15, 256, 3, 2, 1)])
def test_conv_fwd_tile_variants_bf16(cfg):
    """Repeated forward + data-gradient calls of the implicit-GEMM convolution
    at ResNet layer-3/4 widths (the stride-1 dgrad reads the forward weights in
    place; the stride-2 one runs as phase convolutions; later calls run after
    the autotuner settled): every call's output and dx vs the oracle on the
    same bf16 inputs (1e-2).  (A BN = 128 tile for K ≥ 256 was measured 30 %
    slower than BN = 256 on every C4 shape and is not a candidate.)"""
    be = be_init()
    be.set_compute_dtype("bf16")
    N, C, H, W, K, R, st, pd = cfg
    rng = np.random.default_rng(sum(cfg) + 11)
    from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
    q = lambda a: bf16_bits_to_f32(f32_to_bf16_bits(a.astype(np.float32)))
    x = q(rng.standard_normal((N, C, H, W)))
    w = q(rng.standard_normal((K, C, R, R)) / np.sqrt(C * R * R))
    xo, wo = Var(x.astype(np.float64), True), Var(w.astype(np.float64))
    yo = oops.conv2d(xo, wo, None, st, pd)
    g = q(rng.standard_normal(yo.value.shape))
    backward(yo, g.astype(np.float64))
    for _ in range(4):
        xd = be.tensor(nchw_to_nhwc(x), requires_grad=True)
        yd = be.conv2d(be.cast(xd, "bf16"), be.tensor(nchw_to_nhwc(w)), None, st, pd)
        assert rel(nhwc_to_nchw(yd.numpy()), yo.value) < 1e-2
        yd.backward(be.tensor(nchw_to_nhwc(g), dtype="bf16"))
        assert rel(nhwc_to_nchw(xd.grad.numpy()), xo.grad) < 1e-2
