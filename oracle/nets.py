"""ORACLE — test infrastructure only (see oracle/autograd.py header).

The benchmark networks of the paper's Table 1 as plain
float64 compositions of oracle/ops.py, in logical layouts.  Architectures
follow SURVEY.md §8(c) readings 1, 9, 10, 11.  Parameter specs are
(name, shape, init, fan_in) for synth.make_params; Linear weights are
[in, out] (Listing 1), conv weights KCRS.
"""
from __future__ import annotations

import numpy as np

from . import ops
from .autograd import Var


def _lin(name, i, o, bias=True):
    s = [(name + ".w", (i, o), "normal", i)]
    if bias:
        s.append((name + ".b", (o,), "normal", i))
    return s


def _conv(name, k, c, r, bias):
    s = [(name + ".w", (k, c, r, r), "normal", c * r * r)]
    if bias:
        s.append((name + ".b", (k,), "normal", c * r * r))
    return s


def _bn(name, c):
    return [(name + ".g", (c,), "ones", 1), (name + ".b", (c,), "zeros", 1)]


# ---------------------------------------------------------------- MLPs (C1, C2)
class MLP:
    """Stack of Listing-1 LinearLayers with ReLU between them, softmax-CE on
    top.  C1 = MLP((784,128,10)); C2 = MLP((4096,4096,4096,1000))."""

    def __init__(self, sizes):
        self.sizes = tuple(sizes)

    def param_specs(self):
        s = []
        for i in range(len(self.sizes) - 1):
            s += _lin(f"fc{i}", self.sizes[i], self.sizes[i + 1])
        return s

    def logits(self, P, x):
        h = x
        L = len(self.sizes) - 1
        for i in range(L):
            h = ops.linear(h, P[f"fc{i}.w"], P[f"fc{i}.b"])
            if i < L - 1:
                h = ops.relu(h)
        return h

    def loss(self, P, batch, state=None):
        x, y = batch
        z = self.logits(P, Var(x))
        return ops.softmax_cross_entropy(z, y), {"logits": z.value}


# ---------------------------------------------------------------- Listing 1
class ListingNet:
    """Listing 1 FullBasicModel under SURVEY §8(c)
    reading 1: conv(1→128, 3) → ReLU → global avgpool → Linear(128,10) →
    softmax(-CE)."""

    def param_specs(self):
        return _conv("conv", 128, 1, 3, True) + _lin("fc", 128, 10)

    def loss(self, P, batch, state=None):
        x, y = batch
        t1 = ops.conv2d(Var(x), P["conv.w"], P["conv.b"], 1, 0)
        t2 = ops.relu(t1)
        t3 = ops.linear(ops.avgpool_global(t2), P["fc.w"], P["fc.b"])
        return ops.softmax_cross_entropy(t3, y), {"logits": t3.value}


# ---------------------------------------------------------------- AlexNet (C3)
class AlexNet:
    """Single-tower AlexNet (SURVEY §8(c) reading 10): no LRN, dropout p=0,
    adaptive 6×6 pool is the identity at 224²."""
    CONVS = [  # name, K, C, R, stride, pad, pool_after
        ("conv1", 64, 3, 11, 4, 2, True),
        ("conv2", 192, 64, 5, 1, 2, True),
        ("conv3", 384, 192, 3, 1, 1, False),
        ("conv4", 256, 384, 3, 1, 1, False),
        ("conv5", 256, 256, 3, 1, 1, True),
    ]

    def __init__(self, classes=1000, width=1.0, image=224):
        self.classes = classes
        self.image = image
        # width < 1 shrinks every channel count (tiny parity cases only)
        chain, prev = [], 3
        for (n, k, _, r, s, p, pool) in self.CONVS:
            k = max(1, int(k * width))
            chain.append((n, k, prev, r, s, p, pool))
            prev = k
        self.convs = chain
        hw = image
        for (_, _, _, r, s, p, pool) in chain:
            hw = ops.conv_out_size(hw, r, s, p)
            if pool:
                hw = ops.conv_out_size(hw, 3, 2, 0)
        self.feat = prev * hw * hw
        self.fc_hidden = max(1, int(4096 * width))

    def param_specs(self):
        s = []
        for (n, k, c, r, st, p, pool) in self.convs:
            s += _conv(n, k, c, r, True)
        s += _lin("fc6", self.feat, self.fc_hidden)
        s += _lin("fc7", self.fc_hidden, self.fc_hidden)
        s += _lin("fc8", self.fc_hidden, self.classes)
        return s

    def loss(self, P, batch, state=None):
        x, y = batch
        h = Var(x)
        argmaxes = {}
        for (n, k, c, r, st, p, pool) in self.convs:
            h = ops.relu(ops.conv2d(h, P[n + ".w"], P[n + ".b"], st, p))
            if pool:
                h, am = ops.maxpool2d(h, 3, 2, 0)
                argmaxes[n] = am
        h = ops.flatten(h)
        h = ops.relu(ops.linear(h, P["fc6.w"], P["fc6.b"]))
        h = ops.relu(ops.linear(h, P["fc7.w"], P["fc7.b"]))
        z = ops.linear(h, P["fc8.w"], P["fc8.b"])
        return ops.softmax_cross_entropy(z, y), {"logits": z.value, "argmax": argmaxes}


# ---------------------------------------------------------------- ResNet-50 (C4)
class ResNet50:
    """ResNet-50 v1.5 (stride on the 3×3 conv; SURVEY §8(c) reading 9).
    `layers`/`width` shrink it for tiny parity cases; defaults are the real
    net (25,557,032 parameters)."""

    def __init__(self, layers=(3, 4, 6, 3), base=64, classes=1000):
        self.layers = tuple(layers)
        self.base = base
        self.classes = classes

    def blocks(self):
        out = []
        cin = self.base
        for li, nb in enumerate(self.layers):
            mid = self.base * (2 ** li)
            cout = mid * 4
            for bi in range(nb):
                stride = 2 if (bi == 0 and li > 0) else 1
                down = bi == 0
                out.append((f"l{li + 1}.{bi}", cin, mid, cout, stride, down))
                cin = cout
        return out

    def param_specs(self):
        s = _conv("conv1", self.base, 3, 7, False) + _bn("bn1", self.base)
        for (n, cin, mid, cout, stride, down) in self.blocks():
            s += _conv(n + ".c1", mid, cin, 1, False) + _bn(n + ".bn1", mid)
            s += _conv(n + ".c2", mid, mid, 3, False) + _bn(n + ".bn2", mid)
            s += _conv(n + ".c3", cout, mid, 1, False) + _bn(n + ".bn3", cout)
            if down:
                s += _conv(n + ".ds", cout, cin, 1, False) + _bn(n + ".dsbn", cout)
        s += _lin("fc", self.blocks()[-1][3], self.classes)
        return s

    def loss(self, P, batch, state=None):
        x, y = batch
        stats = {}

        def bn(h, name):
            o, st = ops.batchnorm2d(h, P[name + ".g"], P[name + ".b"])
            stats[name] = st
            return o
        h = ops.conv2d(Var(x), P["conv1.w"], None, 2, 3)
        h = ops.relu(bn(h, "bn1"))
        h, am = ops.maxpool2d(h, 3, 2, 1)
        for (n, cin, mid, cout, stride, down) in self.blocks():
            idn = h
            t = ops.relu(bn(ops.conv2d(h, P[n + ".c1.w"], None, 1, 0), n + ".bn1"))
            t = ops.relu(bn(ops.conv2d(t, P[n + ".c2.w"], None, stride, 1), n + ".bn2"))
            t = bn(ops.conv2d(t, P[n + ".c3.w"], None, 1, 0), n + ".bn3")
            if down:
                idn = bn(ops.conv2d(h, P[n + ".ds.w"], None, stride, 0), n + ".dsbn")
            h = ops.relu(ops.add(t, idn))
        h = ops.avgpool_global(h)
        z = ops.linear(h, P["fc.w"], P["fc.b"])
        return ops.softmax_cross_entropy(z, y), {"logits": z.value, "bn_stats": stats,
                                                 "argmax": {"maxpool": am}}


# ---------------------------------------------------------------- NCF (C5)
class NCF:
    """NeuMF (reading 11): GMF (dim 64) and MLP towers
    (128+128 → 256 → 128 → 64, ReLU), head on concat(gmf, mlp) → 1 logit,
    binary loss as 2-class CE on [0, z]."""

    def __init__(self, n_users=138493, n_items=26744, gmf=64, mlp=(256, 256, 128, 64)):
        self.n_users, self.n_items, self.gmf, self.mlp = n_users, n_items, gmf, tuple(mlp)

    def param_specs(self):
        e = self.mlp[0] // 2
        s = [("user_gmf", (self.n_users, self.gmf), "normal", 1),
             ("item_gmf", (self.n_items, self.gmf), "normal", 1),
             ("user_mlp", (self.n_users, e), "normal", 1),
             ("item_mlp", (self.n_items, e), "normal", 1)]
        for i in range(len(self.mlp) - 1):
            s += _lin(f"mlp{i}", self.mlp[i], self.mlp[i + 1])
        s += _lin("head", self.gmf + self.mlp[-1], 1)
        return s

    def loss(self, P, batch, state=None):
        users, items, y = batch
        g = ops.mul(ops.embedding(P["user_gmf"], users), ops.embedding(P["item_gmf"], items))
        h = ops.concat([ops.embedding(P["user_mlp"], users), ops.embedding(P["item_mlp"], items)], 1)
        for i in range(len(self.mlp) - 1):
            h = ops.relu(ops.linear(h, P[f"mlp{i}.w"], P[f"mlp{i}.b"]))
        z = ops.linear(ops.concat([g, h], 1), P["head.w"], P["head.b"])
        return ops.bce_as_two_class_ce(z, y), {"logits": z.value}


# ---------------------------------------------------------------- VGG-19 (Table 1)
class VGG19:
    """VGG-19 (Table 1; configuration "E" of Simonyan & Zisserman,
    the torchvision form — DESIGN.md reading R15): sixteen 3×3/1/1 convs with
    bias + ReLU in five stages of 64, 128, 256, 512, 512 channels, each stage
    closed by maxpool 2×2/2; flatten (NCHW order; the adaptive 7×7 pool is the
    identity at 224²); classifier fc6 25088→4096, ReLU, dropout, fc7
    4096→4096, ReLU, dropout, fc8 4096→1000.  Dropout masks are the
    counter-based draws of ops.dropout with (seed, offset = 6 | 7)."""
    STAGES = ((64, 2), (128, 2), (256, 4), (512, 4), (512, 4))

    def __init__(self, classes=1000, width=1.0, image=224, dropout=0.5, seed=0):
        self.classes, self.image, self.p, self.seed = classes, image, dropout, seed
        chain, prev, hw = [], 3, image
        for si, (k, n) in enumerate(self.STAGES):
            k = max(1, int(k * width))
            for j in range(n):
                chain.append((f"conv{si + 1}_{j + 1}", k, prev, j == n - 1))
                prev = k
            hw //= 2
        self.convs, self.feat = chain, prev * hw * hw
        self.hidden = max(1, int(4096 * width))

    def param_specs(self):
        s = []
        for (n, k, c, pool) in self.convs:
            s += _conv(n, k, c, 3, True)
        return s + _lin("fc6", self.feat, self.hidden) + _lin("fc7", self.hidden, self.hidden) + \
            _lin("fc8", self.hidden, self.classes)

    def loss(self, P, batch, state=None):
        x, y = batch
        h = Var(x)
        for (n, k, c, pool) in self.convs:
            h = ops.relu(ops.conv2d(h, P[n + ".w"], P[n + ".b"], 1, 1))
            if pool:
                h, _ = ops.maxpool2d(h, 2, 2, 0)
        h = ops.flatten(h)
        h = ops.dropout(ops.relu(ops.linear(h, P["fc6.w"], P["fc6.b"])), self.p, self.seed, 6)
        h = ops.dropout(ops.relu(ops.linear(h, P["fc7.w"], P["fc7.b"])), self.p, self.seed, 7)
        z = ops.linear(h, P["fc8.w"], P["fc8.b"])
        return ops.softmax_cross_entropy(z, y), {"logits": z.value}


# ---------------------------------------------------------------- MobileNetV2 (Table 1)
class MobileNetV2:
    """MobileNet (Table 1) read as MobileNetV2 (Sandler et al.
    2018, the torchvision model; reading R13): stem conv 3×3/2
    3→32 + BN + ReLU6; inverted residual blocks (t, c, n, s) =
    (1,16,1,1) (6,24,2,2) (6,32,3,2) (6,64,4,2) (6,96,3,1) (6,160,3,2)
    (6,320,1,1): [1×1 expand + BN + ReLU6 when t > 1] → 3×3 depthwise
    (stride s on the first block of a group) + BN + ReLU6 → 1×1 project + BN,
    plus the identity when stride 1 and C_in = C_out; head 1×1 → 1280 + BN +
    ReLU6; global avgpool; dropout(p); Linear(1280, classes).  Convs have no
    bias.  3,504,872 parameters at the defaults."""
    SETTINGS = ((1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2), (6, 96, 3, 1), (6, 160, 3, 2),
                (6, 320, 1, 1))

    def __init__(self, classes=1000, width=1.0, dropout=0.2, seed=0, settings=None):
        self.classes, self.p, self.seed = classes, dropout, seed
        w = lambda c: max(8, int(c * width))  # noqa: E731
        self.stem = w(32)
        self.last = max(1280, w(1280)) if width >= 1.0 else w(1280)
        blocks, cin = [], self.stem
        for gi, (t, c, n, s) in enumerate(settings or self.SETTINGS):
            cout = w(c)
            for j in range(n):
                blocks.append((f"b{len(blocks)}", cin, cin * t, cout, s if j == 0 else 1, t))
                cin = cout
        self.blocks, self.cfinal = blocks, cin

    def param_specs(self):
        s = _conv("stem", self.stem, 3, 3, False) + _bn("stem_bn", self.stem)
        for (n, cin, hid, cout, st, t) in self.blocks:
            if t != 1:
                s += _conv(n + ".exp", hid, cin, 1, False) + _bn(n + ".exp_bn", hid)
            s += [(n + ".dw.w", (hid, 1, 3, 3), "normal", 9)] + _bn(n + ".dw_bn", hid)
            s += _conv(n + ".proj", cout, hid, 1, False) + _bn(n + ".proj_bn", cout)
        s += _conv("head", self.last, self.cfinal, 1, False) + _bn("head_bn", self.last)
        return s + _lin("fc", self.last, self.classes)

    def loss(self, P, batch, state=None):
        x, y = batch

        def bn(h, name):
            o, _ = ops.batchnorm2d(h, P[name + ".g"], P[name + ".b"])
            return o
        h = ops.relu6(bn(ops.conv2d(Var(x), P["stem.w"], None, 2, 1), "stem_bn"))
        for (n, cin, hid, cout, st, t) in self.blocks:
            u = h
            if t != 1:
                u = ops.relu6(bn(ops.conv2d(u, P[n + ".exp.w"], None, 1, 0), n + ".exp_bn"))
            u = ops.relu6(bn(ops.conv2d_depthwise(u, P[n + ".dw.w"], st, 1), n + ".dw_bn"))
            u = bn(ops.conv2d(u, P[n + ".proj.w"], None, 1, 0), n + ".proj_bn")
            h = ops.add(u, h) if (st == 1 and cin == cout) else u
        h = ops.relu6(bn(ops.conv2d(h, P["head.w"], None, 1, 0), "head_bn"))
        h = ops.dropout(ops.avgpool_global(h), self.p, self.seed, 0)
        z = ops.linear(h, P["fc.w"], P["fc.b"])
        return ops.softmax_cross_entropy(z, y), {"logits": z.value}
