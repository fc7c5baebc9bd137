"""The benchmark networks of the paper's Table 1 written
as eager user programs over the be_* ops (the "models are just Python
programs" stance of PAPER.md:59-64).  Each op call launches device kernels
and records itself on the tape; `loss.backward()` replays the tape in C++.

Device layouts: activations NHWC, conv weights KRSC, Linear weights
[in, out] (Listing 1).  The first conv's input channels are
zero-padded to 8 so every GEMM operand row is 16-B aligned for TMA; the
pad channels' weights start at 0 and stay 0 (their gradient is exactly 0).
AlexNet's fc6 rows are stored in NHWC-flatten order.  `to_device_layout` /
`to_logical_layout` convert parameters at upload / for comparison — host
marshalling only, never on the step path.
"""
from __future__ import annotations

import numpy as np

from . import api as T

CPAD = 8  # first-layer channel padding


def _lin_spec(name, i, o, bias=True):
    s = [(name + ".w", (i, o), "normal", i)]
    if bias:
        s.append((name + ".b", (o,), "normal", i))
    return s


def _conv_spec(name, k, c, r, bias):
    s = [(name + ".w", (k, c, r, r), "normal", c * r * r)]
    if bias:
        s.append((name + ".b", (k,), "normal", c * r * r))
    return s


def _bn_spec(name, c):
    return [(name + ".g", (c,), "ones", 1), (name + ".b", (c,), "zeros", 1)]


def images_to_device(x_nchw: np.ndarray, dtype="bf16", cpad=CPAD) -> T.Tensor:
    """Logical NCHW float32 images → device NHWC with channels padded."""
    N, C, H, W = x_nchw.shape
    nhwc = np.zeros((N, H, W, max(C, cpad)), np.float32)
    nhwc[..., :C] = x_nchw.transpose(0, 2, 3, 1)
    return T.tensor(nhwc, dtype=dtype)


class Model:
    """Parameter registry in deterministic registration order."""

    def __init__(self):
        self.params: dict[str, T.Tensor] = {}
        self.buffers: dict[str, T.Tensor] = {}

    def param_specs(self):
        raise NotImplementedError

    def to_device_layout(self, name, a):
        return a

    def to_logical_layout(self, name, a):
        return a

    def load(self, logical: dict):
        self.params = {}
        for (name, shape, _, _) in self.param_specs():
            self.params[name] = T.tensor(self.to_device_layout(name, np.asarray(logical[name], np.float32)),
                                         requires_grad=True)
        self.make_buffers()
        return self

    def make_buffers(self):
        pass

    def parameters(self):
        return list(self.params.values())

    def embedding_tables(self):
        return []

    def logical(self, name, device_array):
        return self.to_logical_layout(name, device_array)


# ---------------------------------------------------------------- MLP (C1, C2)
class MLP(Model):
    def __init__(self, sizes):
        super().__init__()
        self.sizes = tuple(sizes)

    def param_specs(self):
        s = []
        for i in range(len(self.sizes) - 1):
            s += _lin_spec(f"fc{i}", self.sizes[i], self.sizes[i + 1])
        return s

    def loss(self, x, y):
        h = x
        L = len(self.sizes) - 1
        P = self.params
        for i in range(L):
            last = i == L - 1
            h = T.linear(h, P[f"fc{i}.w"], P[f"fc{i}.b"], act=0 if last else 1, out_f32=last)
        return T.softmax_xent(h, y)


# ---------------------------------------------------------------- Listing 1
class ListingNet(Model):
    """Listing 1 FullBasicModel under the reading conv → ReLU → global
    avgpool → Linear(128,10) → softmax-CE (SURVEY §8(c) reading 1)."""

    def param_specs(self):
        return _conv_spec("conv", 128, 1, 3, True) + _lin_spec("fc", 128, 10)

    def to_device_layout(self, name, a):
        return _conv_to_krsc(a, pad_c=True) if name == "conv.w" else a

    def to_logical_layout(self, name, a):
        return _krsc_to_conv(a, 1) if name == "conv.w" else a

    def loss(self, x, y):
        P = self.params
        t = T.conv2d(x, P["conv.w"], P["conv.b"], 1, 0, act=1)
        t = T.avgpool_global(t)
        z = T.linear(t, P["fc.w"], P["fc.b"], out_f32=True)
        return T.softmax_xent(z, y)


def _conv_to_krsc(w, pad_c=False):
    k = np.ascontiguousarray(np.asarray(w, np.float32).transpose(0, 2, 3, 1))
    if pad_c and k.shape[3] < CPAD:
        z = np.zeros(k.shape[:3] + (CPAD,), np.float32)
        z[..., :k.shape[3]] = k
        k = z
    return k


def _krsc_to_conv(w, c_logical=None):
    w = np.asarray(w)
    if c_logical is not None:
        w = w[..., :c_logical]
    return np.ascontiguousarray(w.transpose(0, 3, 1, 2))


# ---------------------------------------------------------------- AlexNet (C3)
class AlexNet(Model):
    CONVS = [("conv1", 64, 11, 4, 2, True), ("conv2", 192, 5, 1, 2, True), ("conv3", 384, 3, 1, 1, False),
             ("conv4", 256, 3, 1, 1, False), ("conv5", 256, 3, 1, 1, True)]

    def __init__(self, classes=1000, width=1.0, image=224):
        super().__init__()
        self.classes = classes
        chain, prev, hw = [], 3, image
        for (n, k, r, s, p, pool) in self.CONVS:
            k = max(1, int(k * width))
            chain.append((n, k, prev, r, s, p, pool))
            prev = k
            hw = (hw + 2 * p - r) // s + 1
            if pool:
                hw = (hw - 3) // 2 + 1
        self.convs, self.c5, self.hw = chain, prev, hw
        self.hidden = max(1, int(4096 * width))

    def param_specs(self):
        s = []
        for (n, k, c, r, st, p, pool) in self.convs:
            s += _conv_spec(n, k, c, r, True)
        f = self.c5 * self.hw * self.hw
        return s + _lin_spec("fc6", f, self.hidden) + _lin_spec("fc7", self.hidden, self.hidden) + \
            _lin_spec("fc8", self.hidden, self.classes)

    def _fc6_perm(self):
        # device row (h, w, c) ← logical row c·HW + h·W + w
        C, H = self.c5, self.hw
        h, w, c = np.meshgrid(np.arange(H), np.arange(H), np.arange(C), indexing="ij")
        return (c * H * H + h * H + w).reshape(-1)

    def to_device_layout(self, name, a):
        if name.endswith(".w") and name.startswith("conv"):
            return _conv_to_krsc(a, pad_c=(name == "conv1.w"))
        if name == "fc6.w":
            return np.ascontiguousarray(a[self._fc6_perm()])
        return a

    def to_logical_layout(self, name, a):
        if name.endswith(".w") and name.startswith("conv"):
            return _krsc_to_conv(a, 3 if name == "conv1.w" else None)
        if name == "fc6.w":
            out = np.empty_like(a)
            out[self._fc6_perm()] = a
            return out
        return a

    def loss(self, x, y):
        P = self.params
        h = x
        for (n, k, c, r, st, p, pool) in self.convs:
            h = T.conv2d(h, P[n + ".w"], P[n + ".b"], st, p, act=1)
            if pool:
                h = T.maxpool2d(h, 3, 2, 0)
        N = h.shape[0]
        h = T.reshape(h, (N, -1))  # NHWC flatten (fc6 rows stored to match)
        h = T.linear(h, P["fc6.w"], P["fc6.b"], act=1)
        h = T.linear(h, P["fc7.w"], P["fc7.b"], act=1)
        z = T.linear(h, P["fc8.w"], P["fc8.b"], out_f32=True)
        return T.softmax_xent(z, y)


# ---------------------------------------------------------------- ResNet-50 (C4)
class ResNet50(Model):
    """ResNet-50 v1.5 (SURVEY §8(c) reading 9); `layers`/`base` shrink it.
    bn_stats=True (default) takes the BN statistics from the conv epilogues
    (bn1 / bn2 / stem: the convs with R·S·C ≥ K; the expansions keep the
    streaming statistics pass): the column sums are read back from the bf16
    TMA-store staging tile, and the layer-1 3×3 shared-patch kernel carries
    them too — C4 +0.7 % over the separate statistics pass."""

    def __init__(self, layers=(3, 4, 6, 3), base=64, classes=1000, bn_stats=True, fuse_bn_conv=False,
                 fuse_shortcut_bn=True):
        super().__init__()
        self.layers, self.base, self.classes = tuple(layers), base, classes
        self.bn_stats = bn_stats
        # fuse_shortcut_bn (bf16): projection blocks' output relu(bn3 + dsbn(ds)) in one
        # pass (api.batchnorm2d_add_bn)
        self.fuse_shortcut_bn = fuse_shortcut_bn
        # fuse_bn_conv=True: bn2 + ReLU applied inside c3's operand load
        # (BE_OP_BN_CONV1X1, bf16 mode) — the bn2 output never reaches HBM and
        # the step needs 0.7 GB less memory, but the two transform warps throttle
        # the GEMM mainloop: measured C4 11.4k → 9.2k img/s, so off by default
        self.fuse_bn_conv = fuse_bn_conv

    def blocks(self):
        out, cin = [], self.base
        for li, nb in enumerate(self.layers):
            mid = self.base * (2 ** li)
            for bi in range(nb):
                out.append((f"l{li + 1}.{bi}", cin, mid, mid * 4, 2 if (bi == 0 and li > 0) else 1, bi == 0))
                cin = mid * 4
        return out

    def param_specs(self):
        s = _conv_spec("conv1", self.base, 3, 7, False) + _bn_spec("bn1", self.base)
        for (n, cin, mid, cout, stride, down) in self.blocks():
            s += _conv_spec(n + ".c1", mid, cin, 1, False) + _bn_spec(n + ".bn1", mid)
            s += _conv_spec(n + ".c2", mid, mid, 3, False) + _bn_spec(n + ".bn2", mid)
            s += _conv_spec(n + ".c3", cout, mid, 1, False) + _bn_spec(n + ".bn3", cout)
            if down:
                s += _conv_spec(n + ".ds", cout, cin, 1, False) + _bn_spec(n + ".dsbn", cout)
        return s + _lin_spec("fc", self.blocks()[-1][3], self.classes)

    def to_device_layout(self, name, a):
        if a.ndim == 4:
            return _conv_to_krsc(a, pad_c=(name == "conv1.w"))
        return a

    def to_logical_layout(self, name, a):
        if np.ndim(a) == 4:
            return _krsc_to_conv(a, 3 if name == "conv1.w" else None)
        return a

    def make_buffers(self):
        self.buffers = {}
        for (name, shape, init, _) in self.param_specs():
            if name.endswith(".g"):
                base = name[:-2]
                self.buffers[base + ".rm"] = T.tensor(np.zeros(shape, np.float32))
                self.buffers[base + ".rv"] = T.tensor(np.ones(shape, np.float32))

    def loss(self, x, y):
        P, B = self.params, self.buffers

        def bn(h, name, act, residual=None):
            return T.batchnorm2d(h, P[name + ".g"], P[name + ".b"], B[name + ".rm"], B[name + ".rv"], act=act,
                                 residual=residual)
        def conv(h, w, stride, pad):  # every conv feeds a BN (epilogue statistics: self.bn_stats)
            return T.conv2d(h, P[w], None, stride, pad, bn_stats=self.bn_stats)
        h = conv(x, "conv1.w", 2, 3)
        h = bn(h, "bn1", 1)
        h = T.maxpool2d(h, 3, 2, 1)
        fuse = self.fuse_bn_conv and x.dtype == T.L.BE_BF16 and not self.bn_stats
        fuse_sc = self.fuse_shortcut_bn and x.dtype == T.L.BE_BF16
        for (n, cin, mid, cout, stride, down) in self.blocks():
            # the projection shortcut first: the engine runs the later-recorded
            # c1 branch's backward first, so c1's dgrad writes dL/dh in full
            # (beta 0) and the stride-2 projection's phase dgrad only adds into
            # its one live phase (no zero fill of the other three)
            yds = conv(h, n + ".ds.w", stride, 0) if down else None
            idn = None if down and fuse_sc else (bn(yds, n + ".dsbn", 0) if down else h)
            t = bn(conv(h, n + ".c1.w", 1, 0), n + ".bn1", 1)
            t = conv(t, n + ".c2.w", stride, 1)
            if fuse:  # c3(relu(bn2(t))) — the bn2 output is only ever built in c3's operand tiles
                u = T.bn_conv1x1(t, P[n + ".bn2.g"], P[n + ".bn2.b"], B[n + ".bn2.rm"], B[n + ".bn2.rv"],
                                 P[n + ".c3.w"], act=1)
            else:
                u = conv(bn(t, n + ".bn2", 1), n + ".c3.w", 1, 0)
            # block output relu(bn3(c3) + shortcut) in one pass (fused residual BN);
            # projection blocks: relu(bn3(c3) + dsbn(ds)) with the shortcut's BN
            # applied inside that pass (its output never written)
            if idn is None:
                h = T.batchnorm2d_add_bn(u, P[n + ".bn3.g"], P[n + ".bn3.b"], B[n + ".bn3.rm"], B[n + ".bn3.rv"],
                                         yds, P[n + ".dsbn.g"], P[n + ".dsbn.b"], B[n + ".dsbn.rm"],
                                         B[n + ".dsbn.rv"], act=1)
            else:
                h = bn(u, n + ".bn3", 1, residual=idn)
        h = T.avgpool_global(h)
        z = T.linear(h, P["fc.w"], P["fc.b"], out_f32=True)
        return T.softmax_xent(z, y)


# ---------------------------------------------------------------- VGG-19 (Table 1)
class VGG19(Model):
    """VGG-19 (Table 1; oracle/nets.py VGG19, R15):
    sixteen 3×3 convs (bias + ReLU fused into the conv epilogue), 2×2/2
    maxpools, NHWC flatten (fc6 rows stored to match), fc6/fc7 + ReLU +
    counter-based dropout (offsets 6, 7 under `self.seed`), fc8."""
    STAGES = ((64, 2), (128, 2), (256, 4), (512, 4), (512, 4))

    def __init__(self, classes=1000, width=1.0, image=224, dropout=0.5, seed=0):
        super().__init__()
        self.classes, self.p, self.seed = classes, dropout, seed
        chain, prev, hw = [], 3, image
        for si, (k, n) in enumerate(self.STAGES):
            k = max(1, int(k * width))
            for j in range(n):
                chain.append((f"conv{si + 1}_{j + 1}", k, prev, j == n - 1))
                prev = k
            hw //= 2
        self.convs, self.c5, self.hw = chain, prev, hw
        self.hidden = max(1, int(4096 * width))

    def param_specs(self):
        s = []
        for (n, k, c, pool) in self.convs:
            s += _conv_spec(n, k, c, 3, True)
        f = self.c5 * self.hw * self.hw
        return s + _lin_spec("fc6", f, self.hidden) + _lin_spec("fc7", self.hidden, self.hidden) + \
            _lin_spec("fc8", self.hidden, self.classes)

    def _fc6_perm(self):
        C, H = self.c5, self.hw
        h, w, c = np.meshgrid(np.arange(H), np.arange(H), np.arange(C), indexing="ij")
        return (c * H * H + h * H + w).reshape(-1)

    def to_device_layout(self, name, a):
        if name.endswith(".w") and name.startswith("conv"):
            return _conv_to_krsc(a, pad_c=(name == "conv1_1.w"))
        if name == "fc6.w":
            return np.ascontiguousarray(a[self._fc6_perm()])
        return a

    def to_logical_layout(self, name, a):
        if name.endswith(".w") and name.startswith("conv"):
            return _krsc_to_conv(a, 3 if name == "conv1_1.w" else None)
        if name == "fc6.w":
            out = np.empty_like(a)
            out[self._fc6_perm()] = a
            return out
        return a

    def loss(self, x, y):
        P = self.params
        h = x
        for (n, k, c, pool) in self.convs:
            h = T.conv2d(h, P[n + ".w"], P[n + ".b"], 1, 1, act=1)
            if pool:
                h = T.maxpool2d(h, 2, 2, 0)
        h = T.reshape(h, (h.shape[0], -1))
        h = T.dropout(T.linear(h, P["fc6.w"], P["fc6.b"], act=1), self.p, self.seed, 6)
        h = T.dropout(T.linear(h, P["fc7.w"], P["fc7.b"], act=1), self.p, self.seed, 7)
        z = T.linear(h, P["fc8.w"], P["fc8.b"], out_f32=True)
        return T.softmax_xent(z, y)


# ---------------------------------------------------------------- MobileNetV2 (Table 1)
class MobileNetV2(Model):
    """MobileNetV2 (Table 1 "MobileNet"; oracle/nets.py
    MobileNetV2, R13): every conv feeds a batch norm whose ReLU6
    (act = 2) runs in the BN apply pass; 1×1 expand / project convs are
    tcgen05 GEMMs over the NHWC activations, the 3×3 depthwise convs run on
    the depthwise kernels (weights stored RSC); the residual add is fused
    into the projection's BN pass."""
    SETTINGS = ((1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2), (6, 96, 3, 1), (6, 160, 3, 2),
                (6, 320, 1, 1))

    def __init__(self, classes=1000, width=1.0, dropout=0.2, seed=0, settings=None):
        super().__init__()
        self.classes, self.p, self.seed = classes, dropout, seed
        w = lambda c: max(8, int(c * width))  # noqa: E731
        self.stem = w(32)
        self.last = max(1280, w(1280)) if width >= 1.0 else w(1280)
        blocks, cin = [], self.stem
        for (t, c, n, s) in (settings or self.SETTINGS):
            cout = w(c)
            for j in range(n):
                blocks.append((f"b{len(blocks)}", cin, cin * t, cout, s if j == 0 else 1, t))
                cin = cout
        self.blocks, self.cfinal = blocks, cin

    def param_specs(self):
        s = _conv_spec("stem", self.stem, 3, 3, False) + _bn_spec("stem_bn", self.stem)
        for (n, cin, hid, cout, st, t) in self.blocks:
            if t != 1:
                s += _conv_spec(n + ".exp", hid, cin, 1, False) + _bn_spec(n + ".exp_bn", hid)
            s += [(n + ".dw.w", (hid, 1, 3, 3), "normal", 9)] + _bn_spec(n + ".dw_bn", hid)
            s += _conv_spec(n + ".proj", cout, hid, 1, False) + _bn_spec(n + ".proj_bn", cout)
        s += _conv_spec("head", self.last, self.cfinal, 1, False) + _bn_spec("head_bn", self.last)
        return s + _lin_spec("fc", self.last, self.classes)

    def to_device_layout(self, name, a):
        if name.endswith(".dw.w"):
            return np.ascontiguousarray(np.asarray(a, np.float32)[:, 0].transpose(1, 2, 0))  # [C,1,R,S] → RSC
        if np.ndim(a) == 4:
            return _conv_to_krsc(a, pad_c=(name == "stem.w"))
        return a

    def to_logical_layout(self, name, a):
        if name.endswith(".dw.w"):
            return np.ascontiguousarray(np.asarray(a).transpose(2, 0, 1)[:, None])
        if np.ndim(a) == 4:
            return _krsc_to_conv(a, 3 if name == "stem.w" else None)
        return a

    def make_buffers(self):
        self.buffers = {}
        for (name, shape, init, _) in self.param_specs():
            if name.endswith(".g"):
                base = name[:-2]
                self.buffers[base + ".rm"] = T.tensor(np.zeros(shape, np.float32))
                self.buffers[base + ".rv"] = T.tensor(np.ones(shape, np.float32))

    def loss(self, x, y):
        P, B = self.params, self.buffers

        def bn(h, name, act, residual=None):
            return T.batchnorm2d(h, P[name + ".g"], P[name + ".b"], B[name + ".rm"], B[name + ".rv"], act=act,
                                 residual=residual)
        h = bn(T.conv2d(x, P["stem.w"], None, 2, 1), "stem_bn", 2)
        for (n, cin, hid, cout, st, t) in self.blocks:
            u = h
            if t != 1:
                u = bn(T.conv2d(u, P[n + ".exp.w"], None, 1, 0), n + ".exp_bn", 2)
            u = bn(T.conv2d_depthwise(u, P[n + ".dw.w"], st, 1), n + ".dw_bn", 2)
            res = h if (st == 1 and cin == cout) else None
            h = bn(T.conv2d(u, P[n + ".proj.w"], None, 1, 0), n + ".proj_bn", 0, residual=res)
        h = bn(T.conv2d(h, P["head.w"], None, 1, 0), "head_bn", 2)
        h = T.dropout(T.avgpool_global(h), self.p, self.seed, 0)
        z = T.linear(h, P["fc.w"], P["fc.b"], out_f32=True)
        return T.softmax_xent(z, y)


# ---------------------------------------------------------------- NCF (C5)
class NCF(Model):
    """NeuMF (SURVEY §8(c) reading 11): GMF dim 64, MLP 256→256→128→64."""

    def __init__(self, n_users=138493, n_items=26744, gmf=64, mlp=(256, 256, 128, 64)):
        super().__init__()
        self.n_users, self.n_items, self.gmf, self.mlp = n_users, n_items, gmf, tuple(mlp)

    def param_specs(self):
        e = self.mlp[0] // 2
        s = [("user_gmf", (self.n_users, self.gmf), "normal", 1), ("item_gmf", (self.n_items, self.gmf), "normal", 1),
             ("user_mlp", (self.n_users, e), "normal", 1), ("item_mlp", (self.n_items, e), "normal", 1)]
        for i in range(len(self.mlp) - 1):
            s += _lin_spec(f"mlp{i}", self.mlp[i], self.mlp[i + 1])
        return s + _lin_spec("head", self.gmf + self.mlp[-1], 1)

    def embedding_tables(self):
        return [self.params[k] for k in ("user_gmf", "item_gmf", "user_mlp", "item_mlp")]

    def loss(self, users, items, y):
        P = self.params
        g = T.mul(T.embedding(P["user_gmf"], users), T.embedding(P["item_gmf"], items))
        h = T.concat([T.embedding(P["user_mlp"], users), T.embedding(P["item_mlp"], items)])
        for i in range(len(self.mlp) - 1):
            h = T.linear(h, P[f"mlp{i}.w"], P[f"mlp{i}.b"], act=1)
        z = T.linear(T.concat([g, h]), P["head.w"], P["head.b"], out_f32=True)
        return T.bce_logits(z, y)


def train_step(model: Model, batch, lr=0.01, momentum=0.0, weight_decay=0.0, overlap_sgd=False,
               sparse_embeddings=False):
    """One eager step: zero_grad (release), forward, backward, SGD.
    overlap_sgd=False: one fused multi-tensor SGD launch after backward;
    True: each parameter is updated inside backward as soon as its gradient
    is final, on a side stream (be_sgd_overlap) — same values, bitwise.
    sparse_embeddings=True (models with embedding tables): the tables take
    plain SGD (lr, μ = 0, wd = 0) on their touched rows inside the embedding
    backward (be_sgd_sparse); the other parameters as above.
    Returns the (device) loss tensor; nothing here synchronises."""
    tables = model.embedding_tables() if sparse_embeddings else []
    params = [p for p in model.parameters() if all(p is not t for t in tables)]
    key = (lr, momentum, weight_decay, overlap_sgd, bool(tables))
    if getattr(model, "_overlap", None) != key:
        T.sgd_sparse([])
        T.sgd_overlap(params, lr, momentum, weight_decay) if overlap_sgd else T.sgd_overlap([])
        T.sgd_sparse(tables, lr)
        model._overlap = key
    T.zero_grad(params)
    loss = model.loss(*batch)
    loss.backward()
    if not overlap_sgd:
        T.sgd_step(params, lr, momentum, weight_decay)
    if hasattr(model, "seed"):
        model.seed += 1  # a fresh dropout mask every step (counter-based: just a new key)
    return loss
