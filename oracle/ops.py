"""ORACLE — test infrastructure only (see oracle/autograd.py header).

Float64 definitions of every operator on the hot path, each with its
hand-written vector-Jacobian product.  Written as the plain mathematical
definition, no blocking / fusion / reordering beyond the formula.  Layout of
the *logical* tensors: activations NCHW, conv weights KCRS, Linear weights
[in, out] exactly as Listing 1 ("torch.randn(in_sz, out_sz)",
"torch.mm(activations, self.w)").
"""
from __future__ import annotations

import numpy as np

from .autograd import Var, record

f64 = np.float64

def _unbroadcast(g, shape):
    """Sum a broadcast gradient back to `shape` (SPEC S:83-91 right-aligned
    broadcasting; S:278 'broadcasted leaf receives column-summed gradient')."""
    while g.ndim > len(shape):
        g = g.sum(axis=0)
    for i, s in enumerate(shape):
        if s == 1 and g.shape[i] != 1:
            g = g.sum(axis=i, keepdims=True)
    return g


# ---------------------------------------------------------------- elementwise
def add(a: Var, b: Var) -> Var:
    """y = a + b with broadcasting (Listing 1 `t + self.b`, PAPER.md:80;
    residual add y = a + b, both inputs receive dy — SPEC S:312 fan-out)."""
    y = a.value.astype(f64) + b.value.astype(f64)
    sa, sb = a.value.shape, b.value.shape
    return record("add", [a, b], y, lambda g: [_unbroadcast(g, sa), _unbroadcast(g, sb)])


def mul(a: Var, b: Var) -> Var:
    """y = a ⊙ b (NeuMF GMF branch)."""
    av, bv = a.value.astype(f64), b.value.astype(f64)
    return record("mul", [a, b], av * bv,
                  lambda g: [_unbroadcast(g * bv, av.shape), _unbroadcast(g * av, bv.shape)])


def relu(x: Var) -> Var:
    """y = max(x, 0); dx = dy·1[x>0] — gradient 0 at the kink."""
    xv = x.value.astype(f64)
    mask = (xv > 0).astype(f64)
    return record("relu", [x], xv * mask, lambda g: [g * mask])


# ---------------------------------------------------------------- matmul/linear
def matmul(a: Var, b: Var) -> Var:
    """Y = A·B (`torch.mm`); dA = dY·Bᵀ, dB = Aᵀ·dY."""
    av, bv = a.value.astype(f64), b.value.astype(f64)
    return record("matmul", [a, b], av @ bv, lambda g: [g @ bv.T, av.T @ g])


def linear(x: Var, w: Var, b: Var | None) -> Var:
    """Listing 1 LinearLayer.forward: Y = X·W + b.
    dX = dY·Wᵀ, dW = Xᵀ·dY, db = Σ_n dY[n,:]."""
    xv, wv = x.value.astype(f64), w.value.astype(f64)
    y = xv @ wv
    ins = [x, w]
    if b is not None:
        y = y + b.value.astype(f64)[None, :]
        ins.append(b)

    def vjp(g):
        out = [g @ wv.T, xv.T @ g]
        if b is not None:
            out.append(g.sum(axis=0))
        return out
    return record("linear", ins, y, vjp)


def concat(xs, axis=1) -> Var:
    """Column concatenation (NeuMF head input)."""
    vals = [x.value.astype(f64) for x in xs]
    sizes = [v.shape[axis] for v in vals]
    y = np.concatenate(vals, axis=axis)

    def vjp(g):
        return list(np.split(g, np.cumsum(sizes)[:-1], axis=axis))
    return record("concat", list(xs), y, vjp)


def reshape(x: Var, shape) -> Var:
    xs = x.value.shape
    return record("reshape", [x], x.value.astype(f64).reshape(shape), lambda g: [g.reshape(xs)])


def flatten(x: Var) -> Var:
    """Flatten in logical NCHW order: index c·H·W + h·W + w."""
    return reshape(x, (x.value.shape[0], -1))


def sum_all(x: Var) -> Var:
    xs = x.value.shape
    return record("sum", [x], np.asarray(x.value.astype(f64).sum()), lambda g: [np.broadcast_to(g, xs).copy()])


# ---------------------------------------------------------------- convolution
def conv_out_size(H, R, stride, pad):
    """P = floor((H + 2·pad − R)/stride) + 1."""
    return (H + 2 * pad - R) // stride + 1


def im2col_table(N, C, H, W, R, S, stride, pad):
    """The bit-exact "im2col offsets" object T[m, k].

    m = (n, p, q) row-major; k = (r, u, c) row-major (KRSC order);
    h = p·stride − pad + r; w = q·stride − pad + u;
    T = ((n·H + h)·W + w)·C + c, the NHWC offset of the logical input, or −1
    when (h, w) falls in the zero padding.
    """
    P = conv_out_size(H, R, stride, pad)
    Q = conv_out_size(W, S, stride, pad)
    n = np.arange(N, dtype=np.int64)[:, None, None, None, None, None]
    p = np.arange(P, dtype=np.int64)[None, :, None, None, None, None]
    q = np.arange(Q, dtype=np.int64)[None, None, :, None, None, None]
    r = np.arange(R, dtype=np.int64)[None, None, None, :, None, None]
    u = np.arange(S, dtype=np.int64)[None, None, None, None, :, None]
    c = np.arange(C, dtype=np.int64)[None, None, None, None, None, :]
    h = p * stride - pad + r
    w = q * stride - pad + u
    T = ((n * H + h) * W + w) * C + c
    valid = (h >= 0) & (h < H) & (w >= 0) & (w < W)
    T = np.where(valid, T, -1)
    return T.reshape(N * P * Q, R * S * C)


def conv2d(x: Var, w: Var, b: Var | None, stride=1, pad=0, chunk=8) -> Var:
    """Cross-correlation, no kernel flip, zero padding, dilation 1
    (Listing 1 `nn.Conv2d(1, 128, 3)`).

    Y[m, k] = Σ_j gather(X, T)[m, j] · Wmat[k, j] + b[k], Wmat = W in KRSC
    order; dW = dYᵀ·gather(X, T); dX = scatter_add(T, dY·Wmat) skipping −1.
    Evaluated `chunk` images at a time to bound memory (same arithmetic).
    """
    xv = x.value.astype(f64)
    wv = w.value.astype(f64)
    N, C, H, W = xv.shape
    K, C2, R, S = wv.shape
    assert C == C2, "ShapeMismatch"
    P, Q = conv_out_size(H, R, stride, pad), conv_out_size(W, S, stride, pad)
    wmat = wv.transpose(0, 2, 3, 1).reshape(K, R * S * C)          # KRSC
    x_nhwc = np.ascontiguousarray(xv.transpose(0, 2, 3, 1))
    y = np.empty((N, P, Q, K), dtype=f64)
    for n0 in range(0, N, chunk):
        nb = min(chunk, N - n0)
        T = im2col_table(nb, C, H, W, R, S, stride, pad)
        flat = x_nhwc[n0:n0 + nb].reshape(-1)
        cols = np.where(T >= 0, flat[np.maximum(T, 0)], 0.0)
        y[n0:n0 + nb] = (cols @ wmat.T).reshape(nb, P, Q, K)
    if b is not None:
        y = y + b.value.astype(f64)[None, None, None, :]
    y_nchw = np.ascontiguousarray(y.transpose(0, 3, 1, 2))
    ins = [x, w] + ([b] if b is not None else [])

    def vjp(g):
        g_nhwc = g.transpose(0, 2, 3, 1)
        dx = np.zeros(N * H * W * C, dtype=f64)
        dwm = np.zeros((K, R * S * C), dtype=f64)
        for n0 in range(0, N, chunk):
            nb = min(chunk, N - n0)
            T = im2col_table(nb, C, H, W, R, S, stride, pad)
            flat = x_nhwc[n0:n0 + nb].reshape(-1)
            cols = np.where(T >= 0, flat[np.maximum(T, 0)], 0.0)
            gm = g_nhwc[n0:n0 + nb].reshape(nb * P * Q, K)
            dwm += gm.T @ cols
            dcols = gm @ wmat
            m = T >= 0
            dxc = np.zeros(nb * H * W * C, dtype=f64)
            np.add.at(dxc, T[m], dcols[m])
            dx[n0 * H * W * C:(n0 + nb) * H * W * C] = dxc
        dx = dx.reshape(N, H, W, C).transpose(0, 3, 1, 2)
        dw = dwm.reshape(K, R, S, C).transpose(0, 3, 1, 2)
        out = [np.ascontiguousarray(dx), np.ascontiguousarray(dw)]
        if b is not None:
            out.append(g.sum(axis=(0, 2, 3)))
        return out
    return record("conv2d", ins, y_nchw, vjp)


# ---------------------------------------------------------------- pooling
def maxpool2d(x: Var, k=3, stride=2, pad=0):
    """Max pooling with −∞ padding; window scanned row-major (r outer, u
    inner); argmax = FIRST strictly greater element (ties → lowest window
    index; a NaN wins at its first occurrence).  Returns (y, argmax) with
    argmax the int64 plane index h·W + w.
    Backward scatter-adds dy into argmax (windows overlap → accumulate)."""
    xv = x.value.astype(f64)
    N, C, H, W = xv.shape
    P, Q = conv_out_size(H, k, stride, pad), conv_out_size(W, k, stride, pad)
    best = np.full((N, C, P, Q), -np.inf)
    idx = np.full((N, C, P, Q), -1, dtype=np.int64)
    p = np.arange(P)[:, None]
    q = np.arange(Q)[None, :]
    for r in range(k):
        for u in range(k):
            h = p * stride - pad + r
            w = q * stride - pad + u
            valid = (h >= 0) & (h < H) & (w >= 0) & (w < W)          # [P,Q]
            hc, wc = np.clip(h, 0, H - 1), np.clip(w, 0, W - 1)
            val = xv[:, :, hc, wc]                                    # [N,C,P,Q]
            take = valid[None, None] & ((idx < 0) | (val > best) |
                                        (np.isnan(val) & ~np.isnan(best)))
            best = np.where(take, val, best)
            idx = np.where(take, (hc * W + wc)[None, None], idx)

    def vjp(g):
        dx = np.zeros((N * C, H * W), dtype=f64)
        rows = np.repeat(np.arange(N * C), P * Q)
        np.add.at(dx, (rows, idx.reshape(-1)), g.reshape(-1))
        return [dx.reshape(N, C, H, W)]
    y = record("maxpool2d", [x], best, vjp)
    return y, idx


def avgpool_global(x: Var) -> Var:
    """y[n,c] = mean_{h,w} x[n,c,h,w]; dx = dy/(H·W)."""
    xv = x.value.astype(f64)
    N, C, H, W = xv.shape
    return record("avgpool", [x], xv.mean(axis=(2, 3)),
                  lambda g: [np.broadcast_to(g[:, :, None, None] / (H * W), xv.shape).copy()])


# ---------------------------------------------------------------- batch norm
def batchnorm2d(x: Var, gamma: Var, beta: Var, eps=1e-5, momentum=0.1,
                running_mean=None, running_var=None):
    """BatchNorm2d in train mode (PAPER.md:244 names BN; constants per
    SURVEY §8(c)-6 reading): μ, σ² = biased mean/variance over (n,h,w);
    x̂ = (x−μ)/√(σ²+ε); y = γx̂ + β.
    Backward: dβ = Σdy; dγ = Σdy·x̂; dx = γ/√(σ²+ε)·(dy − mean(dy) − x̂·mean(dy·x̂)).
    Running stats (momentum 0.1, unbiased variance) are returned, not used."""
    xv = x.value.astype(f64)
    N, C, H, W = xv.shape
    cnt = N * H * W
    mu = xv.mean(axis=(0, 2, 3))
    var = ((xv - mu[None, :, None, None]) ** 2).mean(axis=(0, 2, 3))
    inv = 1.0 / np.sqrt(var + eps)
    xhat = (xv - mu[None, :, None, None]) * inv[None, :, None, None]
    gv, bv = gamma.value.astype(f64), beta.value.astype(f64)
    y = gv[None, :, None, None] * xhat + bv[None, :, None, None]

    def vjp(g):
        dbeta = g.sum(axis=(0, 2, 3))
        dgamma = (g * xhat).sum(axis=(0, 2, 3))
        mdy = g.mean(axis=(0, 2, 3))[None, :, None, None]
        mdyx = (g * xhat).mean(axis=(0, 2, 3))[None, :, None, None]
        dx = (gv * inv)[None, :, None, None] * (g - mdy - xhat * mdyx)
        return [dx, dgamma, dbeta]
    out = record("batchnorm2d", [x, gamma, beta], y, vjp)
    rm = running_mean if running_mean is not None else np.zeros(C)
    rv = running_var if running_var is not None else np.ones(C)
    new_rm = (1 - momentum) * rm + momentum * mu
    new_rv = (1 - momentum) * rv + momentum * var * cnt / max(cnt - 1, 1)
    return out, (new_rm, new_rv)


# ---------------------------------------------------------------- losses
def softmax(z):
    """Stable softmax over the class axis (dim 1, SURVEY §8(c) reading 2)."""
    z = np.asarray(z, dtype=f64)
    m = z.max(axis=-1, keepdims=True)
    e = np.exp(z - m)
    return e / e.sum(axis=-1, keepdims=True)


def softmax_cross_entropy(z: Var, y: np.ndarray) -> Var:
    """Listing 1's softmax + mean NLL (reduction =
    mean, SURVEY §8(c) reading 4):
    loss = (1/B) Σ_i [max_i + log Σ_j e^{z_ij − max_i} − z_{i,y_i}];
    dz = (softmax(z) − onehot(y))/B."""
    zv = z.value.astype(f64)
    B = zv.shape[0]
    m = zv.max(axis=1)
    lse = m + np.log(np.exp(zv - m[:, None]).sum(axis=1))
    loss = (lse - zv[np.arange(B), y]).sum() / B

    def vjp(g):
        p = softmax(zv)
        p[np.arange(B), y] -= 1.0
        return [g * p / B]
    return record("softmax_xent", [z], np.asarray(loss), vjp)


def argmax_rows(z):
    """First maximum per row (SURVEY §8(c) reading 7)."""
    return np.argmax(np.asarray(z), axis=1).astype(np.int64)


def bce_as_two_class_ce(z: Var, y: np.ndarray) -> Var:
    """NCF's binary loss written as 2-class softmax-CE on logits [0, z]
    (SURVEY §8(c)-9)."""
    B = z.value.shape[0]
    zeros = Var(np.zeros((B, 1)))
    logits = concat([zeros, reshape(z, (B, 1))], axis=1)
    return softmax_cross_entropy(logits, y)


# ---------------------------------------------------------------- embedding
def embedding(table: Var, ids: np.ndarray) -> Var:
    """rows = E[ids]; dE = zeros; np.add.at(dE, ids, dRows)."""
    tv = table.value.astype(f64)

    def vjp(g):
        d = np.zeros_like(tv)
        np.add.at(d, ids, g)
        return [d]
    return record("embedding", [table], tv[ids], vjp)


# ---------------------------------------------------------------- ReLU6 (MobileNetV2)
def relu6(x: Var) -> Var:
    """y = min(max(x, 0), 6); dx = dy·1[0 < x < 6] (gradient 0 at both kinks,
    the ReLU convention of SPEC S:203 extended to the upper clamp).  MobileNetV2's
    activation (Table 1 "MobileNet"; reading R13)."""
    xv = x.value.astype(f64)
    mask = ((xv > 0) & (xv < 6)).astype(f64)
    return record("relu6", [x], np.clip(xv, 0.0, 6.0), lambda g: [g * mask])


# ---------------------------------------------------------------- depthwise convolution
def conv2d_depthwise(x: Var, w: Var, stride=1, pad=0) -> Var:
    """Depthwise convolution (groups = C, one R×S filter per channel; the
    separable convolutions of MobileNet, Table 1):
        y[n,c,p,q] = Σ_{r,s} x[n, c, p·stride − pad + r, q·stride − pad + s] · w[c, 0, r, s]
    with zero padding (cross-correlation, no flip, as conv2d / SPEC S:113-121).
    dx[n,c,h,w] = Σ over the (p,q,r,s) with h = p·stride−pad+r, w = q·stride−pad+s of dy·w;
    dw[c,0,r,s] = Σ_{n,p,q} dy[n,c,p,q] · x[n,c,p·stride−pad+r, q·stride−pad+s]."""
    xv = x.value.astype(f64)
    wv = w.value.astype(f64)
    N, C, H, W = xv.shape
    C2, one, R, S = wv.shape
    assert C == C2 and one == 1, "ShapeMismatch"
    P, Q = conv_out_size(H, R, stride, pad), conv_out_size(W, S, stride, pad)
    xp = np.zeros((N, C, H + 2 * pad + R, W + 2 * pad + S), dtype=f64)
    xp[:, :, pad:pad + H, pad:pad + W] = xv
    y = np.zeros((N, C, P, Q), dtype=f64)
    for r in range(R):
        for s in range(S):
            win = xp[:, :, r:r + stride * (P - 1) + 1:stride, s:s + stride * (Q - 1) + 1:stride]
            y += win * wv[None, :, 0, r, s, None, None]

    def vjp(g):
        dxp = np.zeros_like(xp)
        dw = np.zeros_like(wv)
        for r in range(R):
            for s in range(S):
                win = xp[:, :, r:r + stride * (P - 1) + 1:stride, s:s + stride * (Q - 1) + 1:stride]
                dw[:, 0, r, s] = (g * win).sum(axis=(0, 2, 3))
                dxp[:, :, r:r + stride * (P - 1) + 1:stride, s:s + stride * (Q - 1) + 1:stride] += \
                    g * wv[None, :, 0, r, s, None, None]
        return [np.ascontiguousarray(dxp[:, :, pad:pad + H, pad:pad + W]), dw]
    return record("conv2d_depthwise", [x, w], y, vjp)


# ---------------------------------------------------------------- dropout
_PHILOX_M0, _PHILOX_M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
_PHILOX_W0, _PHILOX_W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
_M64 = (1 << 64) - 1


def _mulhilo64(a, b):
    """(hi, lo) 64-bit halves of the 128-bit product of uint64 arrays a·b,
    from 32-bit limbs (plain schoolbook multiplication)."""
    m32 = np.uint64(0xFFFFFFFF)
    s32 = np.uint64(32)
    a_lo, a_hi = a & m32, a >> s32
    b_lo, b_hi = b & m32, b >> s32
    ll = a_lo * b_lo
    lh = a_lo * b_hi
    hl = a_hi * b_lo
    hh = a_hi * b_hi
    mid = (ll >> s32) + (lh & m32) + (hl & m32)
    lo = (ll & m32) | ((mid & m32) << s32)
    hi = hh + (lh >> s32) + (hl >> s32) + (mid >> s32)
    return hi, lo


def philox4x64_10(counter, key):
    """Philox4x64-10 (Salmon et al., SC'11 "Parallel random numbers: as easy
    as 1, 2, 3"): counter uint64[..., 4], key uint64[2] → uint64[..., 4].
    Each round: (hi0, lo0) = M0·c0, (hi1, lo1) = M1·c2;
    c ← (hi1 ⊕ c1 ⊕ k0, lo1, hi0 ⊕ c3 ⊕ k1, lo0); then the key is bumped by
    the Weyl constants (W0, W1).  Ten rounds."""
    with np.errstate(over="ignore"):
        c = [np.asarray(counter[..., i], dtype=np.uint64).copy() for i in range(4)]
        k0 = np.uint64(int(key[0]) & _M64)
        k1 = np.uint64(int(key[1]) & _M64)
        for rnd in range(10):
            if rnd:
                k0 = np.uint64((int(k0) + _PHILOX_W0) & _M64)
                k1 = np.uint64((int(k1) + _PHILOX_W1) & _M64)
            hi0, lo0 = _mulhilo64(np.uint64(_PHILOX_M0), c[0])
            hi1, lo1 = _mulhilo64(np.uint64(_PHILOX_M1), c[2])
            c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        return np.stack(c, axis=-1)


def dropout_keep_mask(n, p, seed, offset):
    """Keep decisions of dropout for elements i = 0..n-1 (row-major over the
    logical tensor) — a counter-based draw, so the backward pass and every
    replica regenerate it from (seed, offset) alone (reading R14):
      word_i = Philox4x64-10(counter = (i // 4, offset, 0, 0), key = (seed, 0))[i % 4]
      keep_i = (word_i >> 32) >= T,  T = floor(p · 2^32)   (integer compare)."""
    i = np.arange(n, dtype=np.uint64)
    blocks = np.arange((n + 3) // 4, dtype=np.uint64)
    ctr = np.zeros((len(blocks), 4), dtype=np.uint64)
    ctr[:, 0] = blocks
    ctr[:, 1] = np.uint64(int(offset) & _M64)
    words = philox4x64_10(ctr, (seed, 0)).reshape(-1)[:n]
    T = int(np.floor(float(p) * 4294967296.0))
    del i
    return (words >> np.uint64(32)) >= np.uint64(T)


def dropout(x: Var, p: float, seed: int, offset: int = 0, training: bool = True) -> Var:
    """Inverted dropout (Listing 1 / §4.1 names dropout,
    PAPER.md:64): y = x·keep/(1−p) in training, y = x otherwise; dx = dy·keep/(1−p).
    p = 1 drops everything (y = 0)."""
    xv = x.value.astype(f64)
    if not training or p == 0.0:
        return record("dropout", [x], xv.copy(), lambda g: [g])
    keep = dropout_keep_mask(xv.size, p, seed, offset).reshape(xv.shape).astype(f64)
    scale = 0.0 if p >= 1.0 else 1.0 / (1.0 - p)
    return record("dropout", [x], xv * keep * scale, lambda g: [g * keep * scale])
