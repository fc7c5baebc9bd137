"""Teacher-forced, full-depth per-op parity (test infrastructure).

SURVEY §8(c) reading 15: a deep bf16 network's end-to-end gradient error has
no closed form ("parity unpinned"), so every op of the FULL architecture is
gated instead, each fed the device's own inputs:

  1. trace: run the network's eager forward on the device with the api
     functions wrapped; every op call records its attributes and a host copy
     of every input and output tensor (the device's own activations);
  2. replay, last op first: re-run the op on the device on fresh leaves
     holding exactly the traced input values, backpropagate the upstream
     gradient the device produced for that op's output, and compute the
     SAME op with the float64 oracle (oracle/ops.py) on the same values;
     compare forward output, every input gradient, and (BN) running
     statistics, element-wise (∞-norm relative, oracle/compare.py) at the
     north_star tolerance (2e-2 bf16, 1e-4 fp32);
  3. the device's input gradients become the upstream of the producing ops
     (fan-out contributions summed).

Integer decisions are compared bit-exactly on identical inputs (max-pool
winners, softmax argmax).  ReLU masks fused into an op are taken from the
device's own output (SURVEY §8(c) reading 16: a decision taken from floating
point is taken from the same value on both sides).  Layout: the device is
NHWC / KRSC; the oracle is NCHW / KCRS; Linear weights are [in, out] on both.
"""
from __future__ import annotations

import inspect

import numpy as np

import synth
from oracle import ops as oops
from oracle.autograd import Var, backward
from oracle.compare import rel_err

F64 = np.float64


def nhwc_to_nchw(a):
    return np.ascontiguousarray(np.asarray(a).transpose(0, 3, 1, 2))


def nchw_to_nhwc(a):
    return np.ascontiguousarray(np.asarray(a).transpose(0, 2, 3, 1))


class _Ref:
    __slots__ = ("key",)

    def __init__(self, key):
        self.key = key

    def __repr__(self):
        return f"<{self.key}>"


class OpTrace:
    """Wraps the api ops a model calls (be.nn uses the module global `T`)."""

    OPS = ("conv2d", "batchnorm2d", "maxpool2d", "avgpool_global", "reshape", "linear", "softmax_xent",
           "embedding", "mul", "concat", "bce_logits", "add_relu", "dropout", "conv2d_depthwise", "bn_conv1x1",
           "batchnorm2d_add_bn")

    def __init__(self, api, model):
        self.api = api
        self.model = model
        self.recs = []
        self.vals = {}       # key -> host value (float32 / int32), device layout
        self.dtypes = {}     # key -> dtype code
        self.keep = []       # keep traced tensors alive (stable ids)
        self.ids = {}
        self.producer = {}   # key -> record index
        for n, p in model.params.items():
            self.ids[id(p)] = ("param", n)
        for n, b in model.buffers.items():
            self.ids[id(b)] = ("buf", n)

    # ------------------------------------------------------------ tracing
    def _key(self, t):
        k = self.ids.get(id(t))
        if k is None:
            k = ("act", len(self.ids))
            self.ids[id(t)] = k
            self.keep.append(t)
        if k not in self.vals:
            self.vals[k] = t.numpy()
            self.dtypes[k] = t.dtype
        return k

    def _wrap(self, name):
        fn = getattr(self.api, name)
        sig = inspect.signature(fn)

        def traced(*args, **kw):
            b = sig.bind(*args, **kw)
            b.apply_defaults()
            a = dict(b.arguments)
            rec_args = {}
            for k, v in a.items():
                if isinstance(v, self.api.Tensor):
                    rec_args[k] = _Ref(self._key(v))
                elif isinstance(v, (list, tuple)) and v and isinstance(v[0], self.api.Tensor):
                    rec_args[k] = [_Ref(self._key(t)) for t in v]
                else:
                    rec_args[k] = v
            extra = None
            if name in ("maxpool2d", "softmax_xent"):
                a["with_argmax"] = True
                out, am = fn(**a)
                extra = am.numpy()
            else:
                out = fn(**a)
            ok = ("act", len(self.ids))
            self.ids[id(out)] = ok
            self.keep.append(out)
            self.vals[ok] = out.numpy()
            self.dtypes[ok] = out.dtype
            self.producer[ok] = len(self.recs)
            self.recs.append(dict(op=name, args=rec_args, out=ok, extra=extra))
            return out
        return traced

    def install(self, nn_module):
        class Proxy:
            pass
        proxy = Proxy()
        for n in dir(self.api):
            if not n.startswith("__"):
                setattr(proxy, n, getattr(self.api, n))
        for n in self.OPS:
            if hasattr(self.api, n):
                setattr(proxy, n, self._wrap(n))
        self._saved = nn_module.T
        nn_module.T = proxy
        return self

    def uninstall(self, nn_module):
        nn_module.T = self._saved


# ------------------------------------------------------------------ replay
def _leaf(be, val, dt, requires_grad):
    """Fresh device leaf holding exactly `val`; bf16 values go through a
    differentiable cast of an f32 leaf (bf16→f32 gradient widening is exact)."""
    if dt == be._lib.BE_BF16:
        base = be.tensor(val.astype(np.float32), requires_grad=requires_grad)
        return base, be.cast(base, "bf16")
    if dt in (be._lib.BE_I32, be._lib.BE_I64, be._lib.BE_U8):
        t = be.tensor(val)
        return t, t
    t = be.tensor(val.astype(np.float32), requires_grad=requires_grad)
    return t, t


def _as_dtype_values(be, g, dt):
    g = np.asarray(g, np.float32)
    return synth.bf16_values(g) if dt == be._lib.BE_BF16 else g


def _act(v, act):
    """Fused activation of a BN / conv: 1 ReLU, 2 ReLU6 (oracle relu / relu6)."""
    if act == 2:
        return np.clip(v, 0.0, 6.0)
    return np.maximum(v, 0) if act else v


def _act_mask(y, act):
    """The mask the device's backward takes, decided from the device's own
    output (SURVEY §8(c) reading 16): ReLU 1[y > 0]; ReLU6 1[0 < y < 6]."""
    return ((y > 0) & (y < 6)) if act == 2 else (y > 0)


class Replay:
    def __init__(self, be, trace: OpTrace, tol: float, param_logical=None):
        self.be = be
        self.tr = trace
        self.tol = tol
        self.errs = []          # (record idx, op, what, err)
        self.grads = {}         # key -> float64 accumulated upstream (device layout)
        self.param_grads = {}   # param name -> device per-op grads summed (device layout)

    def _upstream(self, key):
        return self.grads.get(key)

    def _push(self, key, g):
        if key[0] == "act" and key not in self.tr.producer:
            return  # a network input (no producer): nothing upstream
        if key[0] == "param":
            self.param_grads[key[1]] = self.param_grads.get(key[1], 0) + np.asarray(g, F64)
            return
        if key[0] == "buf":
            return
        self.grads[key] = self.grads.get(key, 0) + np.asarray(g, F64)

    def record(self, i, op, what, dev, orc, exact=False, mass=None):
        """exact: bit-exact (integer decisions).  mass: the tensor is a
        per-channel SUM Σ_i t_ic whose terms may cancel (BN dβ, dγ, running
        mean); its error is taken against the sum's own scale
        max_c Σ_i |t_ic| — Higham's forward-error bound of summation,
        |ŝ − s| ≤ γ_n Σ|t_i| — instead of max|o|, which is rounding noise
        when the exact sum is 0 (reading R16: e.g. Σ dy = 0 per
        channel behind a conv → BN path)."""
        if exact:
            e = 0.0 if np.array_equal(np.asarray(dev), np.asarray(orc)) else float("inf")
        elif mass is not None:
            d = np.abs(np.asarray(dev, F64) - np.asarray(orc, F64)).max() if np.size(orc) else 0.0
            e = float(d / max(np.abs(np.asarray(orc, F64)).max(), float(mass), 1e-300))
        else:
            e = rel_err(dev, orc)
        self.errs.append((i, op, what, e))

    def run(self):
        be = self.be
        for i in reversed(range(len(self.tr.recs))):
            rec = self.tr.recs[i]
            getattr(self, "_op_" + rec["op"])(i, rec)
        return self

    # ------------------------------------------------------------ helpers
    def _val(self, r):
        return self.tr.vals[r.key]

    def _dt(self, r):
        return self.tr.dtypes[r.key]

    def _req(self, r):
        return r.key[0] == "param" or (r.key[0] == "act" and r.key in self.tr.producer)

    def _dev_inputs(self, rec, names):
        """Fresh leaves for the named tensor args: {name: (leaf, operand)}."""
        out = {}
        for n in names:
            r = rec["args"].get(n)
            if r is None:
                out[n] = (None, None)
            elif isinstance(r, list):
                out[n] = [_leaf(self.be, self._val(x), self._dt(x), self._req(x)) for x in r]
            else:
                out[n] = _leaf(self.be, self._val(r), self._dt(r), self._req(r))
        return out

    def _g_out(self, rec):
        g = self.grads.pop(rec["out"], None)
        return g

    def _dev_backward(self, out, g, rec):
        be = self.be
        if g is None:
            return False
        dt = self.tr.dtypes[rec["out"]]
        if np.ndim(g) == 0 and out.numel() == 1 and dt == be._lib.BE_F32 and float(g) == 1.0:
            out.backward()
        else:
            gv = _as_dtype_values(be, np.asarray(g).reshape(out.shape), dt)
            out.backward(be.tensor(gv, dtype="bf16" if dt == be._lib.BE_BF16 else None))
        return True

    def _finish(self, i, rec, leaves, orc_grads, names, to_dev=None, masses=None):
        """Compare device leaf grads with oracle grads (both device layout) and push upstream."""
        for n in names:
            r = rec["args"].get(n)
            if r is None or not self._req(r):
                continue
            leaf = leaves[n][0]
            gd = leaf.grad.numpy() if leaf.grad is not None else np.zeros_like(self._val(r))
            go = orc_grads[n]
            self.record(i, rec["op"], "d" + n + (":" + r.key[1] if r.key[0] == "param" else ""), gd, go,
                        mass=(masses or {}).get(n))
            self._push(r.key, gd)

    # ------------------------------------------------------------ ops
    def _op_conv2d(self, i, rec):
        be, a = self.be, rec["args"]
        L = self._dev_inputs(rec, ["x", "w", "b"])
        y = be.conv2d(L["x"][1], L["w"][1], L["b"][1], a["stride"], a["pad"], act=a["act"], out_f32=a["out_f32"])
        x = nhwc_to_nchw(self._val(a["x"])).astype(F64)
        w = nhwc_to_nchw(self._val(a["w"])).astype(F64)      # KRSC -> KCRS
        xo, wo = Var(x, True), Var(w, True)
        bo = Var(self._val(a["b"]).astype(F64), True) if a["b"] is not None else None
        zo = oops.conv2d(xo, wo, bo, a["stride"], a["pad"])
        ydev = y.numpy()  # the re-run's own output: its ReLU mask is the one its backward uses
        mask = (nhwc_to_nchw(ydev) > 0) if a["act"] else None
        fwd = np.maximum(zo.value, 0) if a["act"] else zo.value
        self.record(i, "conv2d", "y", nhwc_to_nchw(ydev), fwd)
        g = self._g_out(rec)
        if not self._dev_backward(y, g, rec):
            return
        gn = nhwc_to_nchw(np.asarray(g).reshape(ydev.shape))
        if mask is not None:
            gn = gn * mask
        backward(zo, gn)
        og = {"x": nchw_to_nhwc(xo.grad), "w": nchw_to_nhwc(wo.grad)}
        if bo is not None:
            og["b"] = bo.grad
        self._finish(i, rec, L, og, ["x", "w", "b"])

    def _op_batchnorm2d_add_bn(self, i, rec):
        """act(bn(x) + bn_r(xr)) (the projection block output with the shortcut's
        BN fused into the apply): oracle = the two batchnorm2d's composed."""
        be, a = self.be, rec["args"]
        names = ["x", "gamma", "beta", "xr", "gamma_r", "beta_r"]
        L = self._dev_inputs(rec, names)
        stats = {}
        for sfx in ("", "_r"):
            rm0, rv0 = self._val(a["running_mean" + sfx]), self._val(a["running_var" + sfx])
            stats[sfx] = (rm0, rv0, be.tensor(rm0), be.tensor(rv0))
        y = be.batchnorm2d_add_bn(L["x"][1], L["gamma"][1], L["beta"][1], stats[""][2], stats[""][3],
                                  L["xr"][1], L["gamma_r"][1], L["beta_r"][1], stats["_r"][2], stats["_r"][3],
                                  eps=a["eps"], momentum=a["momentum"], act=a["act"])
        V = {n: Var((nhwc_to_nchw(self._val(a[n])) if n in ("x", "xr") else self._val(a[n])).astype(F64), True)
             for n in names}
        z1, (rm, rv) = oops.batchnorm2d(V["x"], V["gamma"], V["beta"], eps=a["eps"], momentum=a["momentum"],
                                        running_mean=stats[""][0].astype(F64), running_var=stats[""][1].astype(F64))
        z2, (rmr, rvr) = oops.batchnorm2d(V["xr"], V["gamma_r"], V["beta_r"], eps=a["eps"], momentum=a["momentum"],
                                          running_mean=stats["_r"][0].astype(F64),
                                          running_var=stats["_r"][1].astype(F64))
        zo = oops.add(z1, z2)
        ydev = y.numpy()
        self.record(i, "batchnorm2d_add_bn", "y", nhwc_to_nchw(ydev), _act(zo.value, a["act"]))
        for sfx, (rmo, rvo) in (("", (rm, rv)), ("_r", (rmr, rvr))):
            self.record(i, "batchnorm2d_add_bn", "running_mean" + sfx, stats[sfx][2].numpy(), rmo)
            self.record(i, "batchnorm2d_add_bn", "running_var" + sfx, stats[sfx][3].numpy(), rvo)
        g = self._g_out(rec)
        if not self._dev_backward(y, g, rec):
            return
        gn = nhwc_to_nchw(np.asarray(g).reshape(ydev.shape))
        if a["act"]:
            gn = gn * _act_mask(nhwc_to_nchw(ydev), a["act"])
        backward(zo, gn)
        og = {n: (nchw_to_nhwc(V[n].grad) if n in ("x", "xr") else V[n].grad) for n in names}
        masses = {}
        for sfx, xn in (("", "x"), ("_r", "xr")):
            xv = nhwc_to_nchw(self._val(a[xn])).astype(F64)
            xhat = (xv - xv.mean(axis=(0, 2, 3), keepdims=True)) / np.sqrt(xv.var(axis=(0, 2, 3), keepdims=True) + a["eps"])
            masses["beta" + sfx] = np.abs(gn).sum(axis=(0, 2, 3)).max()
            masses["gamma" + sfx] = np.abs(gn * xhat).sum(axis=(0, 2, 3)).max()
        self._finish(i, rec, L, og, names, masses=masses)

    def _op_batchnorm2d(self, i, rec):
        be, a = self.be, rec["args"]
        L = self._dev_inputs(rec, ["x", "gamma", "beta", "residual"])
        rm0 = self._val(a["running_mean"]) if a["running_mean"] is not None else None
        rv0 = self._val(a["running_var"]) if a["running_var"] is not None else None
        rmd = be.tensor(rm0) if rm0 is not None else None
        rvd = be.tensor(rv0) if rv0 is not None else None
        y = be.batchnorm2d(L["x"][1], L["gamma"][1], L["beta"][1], rmd, rvd, eps=a["eps"], momentum=a["momentum"],
                           act=a["act"], residual=L["residual"][1])
        xo = Var(nhwc_to_nchw(self._val(a["x"])).astype(F64), True)
        go = Var(self._val(a["gamma"]).astype(F64), True)
        bo = Var(self._val(a["beta"]).astype(F64), True)
        zo, (rm, rv) = oops.batchnorm2d(xo, go, bo, eps=a["eps"], momentum=a["momentum"],
                                        running_mean=None if rm0 is None else rm0.astype(F64),
                                        running_var=None if rv0 is None else rv0.astype(F64))
        ro = None
        if a["residual"] is not None:
            ro = Var(nhwc_to_nchw(self._val(a["residual"])).astype(F64), True)
            zo = oops.add(zo, ro)
        ydev = y.numpy()
        fwd = _act(zo.value, a["act"])
        self.record(i, "batchnorm2d", "y", nhwc_to_nchw(ydev), fwd)
        if rmd is not None:
            xa = np.abs(nhwc_to_nchw(self._val(a["x"])).astype(F64)).mean(axis=(0, 2, 3))
            rm_mass = (a["momentum"] * xa + (1 - a["momentum"]) * np.abs(rm0)).max()
            self.record(i, "batchnorm2d", "running_mean", rmd.numpy(), rm, mass=rm_mass)
            self.record(i, "batchnorm2d", "running_var", rvd.numpy(), rv)
        g = self._g_out(rec)
        if not self._dev_backward(y, g, rec):
            return
        gn = nhwc_to_nchw(np.asarray(g).reshape(ydev.shape))
        if a["act"]:
            gn = gn * _act_mask(nhwc_to_nchw(ydev), a["act"])
        backward(zo, gn)
        og = {"x": nchw_to_nhwc(xo.grad), "gamma": go.grad, "beta": bo.grad}
        if ro is not None:
            og["residual"] = nchw_to_nhwc(ro.grad)
        xv = nhwc_to_nchw(self._val(a["x"])).astype(F64)
        xhat = (xv - xv.mean(axis=(0, 2, 3), keepdims=True)) / np.sqrt(xv.var(axis=(0, 2, 3), keepdims=True) + a["eps"])
        masses = {"beta": np.abs(gn).sum(axis=(0, 2, 3)).max(), "gamma": np.abs(gn * xhat).sum(axis=(0, 2, 3)).max()}
        self._finish(i, rec, L, og, ["x", "gamma", "beta", "residual"], masses=masses)

    def _op_maxpool2d(self, i, rec):
        be, a = self.be, rec["args"]
        L = self._dev_inputs(rec, ["x"])
        y = be.maxpool2d(L["x"][1], a["k"], a["stride"], a["pad"])
        xv = nhwc_to_nchw(self._val(a["x"])).astype(F64)
        xo = Var(xv, True)
        yo, am = oops.maxpool2d(xo, a["k"], a["stride"], a["pad"])
        ydev = self.tr.vals[rec["out"]]
        self.record(i, "maxpool2d", "y", nhwc_to_nchw(ydev), yo.value)
        # device winner (window index r·k+u, NHWC) → plane index h·W+w: bit-exact
        win = nhwc_to_nchw(rec["extra"]).astype(np.int64)
        P, Q = yo.value.shape[2], yo.value.shape[3]
        hh = np.arange(P)[:, None] * a["stride"] - a["pad"] + win // a["k"]
        ww = np.arange(Q)[None, :] * a["stride"] - a["pad"] + win % a["k"]
        self.record(i, "maxpool2d", "argmax", hh * xv.shape[3] + ww, am, exact=True)
        g = self._g_out(rec)
        if not self._dev_backward(y, g, rec):
            return
        backward(yo, nhwc_to_nchw(np.asarray(g).reshape(ydev.shape)))
        self._finish(i, rec, L, {"x": nchw_to_nhwc(xo.grad)}, ["x"])

    def _op_avgpool_global(self, i, rec):
        be, a = self.be, rec["args"]
        L = self._dev_inputs(rec, ["x"])
        y = be.avgpool_global(L["x"][1])
        xo = Var(nhwc_to_nchw(self._val(a["x"])).astype(F64), True)
        yo = oops.avgpool_global(xo)
        self.record(i, "avgpool", "y", self.tr.vals[rec["out"]], yo.value)
        g = self._g_out(rec)
        if not self._dev_backward(y, g, rec):
            return
        backward(yo, np.asarray(g, F64))
        self._finish(i, rec, L, {"x": nchw_to_nhwc(xo.grad)}, ["x"])

    def _op_reshape(self, i, rec):
        a = rec["args"]
        # a view: values must be identical, the gradient is reshaped back
        self.record(i, "reshape", "y", self.tr.vals[rec["out"]],
                    self._val(a["x"]).reshape(self.tr.vals[rec["out"]].shape), exact=True)
        g = self._g_out(rec)
        if g is not None and self._req(a["x"]):
            self._push(a["x"].key, np.asarray(g).reshape(self._val(a["x"]).shape))

    def _op_linear(self, i, rec):
        be, a = self.be, rec["args"]
        L = self._dev_inputs(rec, ["x", "w", "b"])
        y = be.linear(L["x"][1], L["w"][1], L["b"][1], act=a["act"], out_f32=a["out_f32"])
        xo = Var(self._val(a["x"]).astype(F64), True)
        wo = Var(self._val(a["w"]).astype(F64), True)
        bo = Var(self._val(a["b"]).astype(F64), True) if a["b"] is not None else None
        zo = oops.linear(xo, wo, bo)
        ydev = y.numpy()
        fwd = np.maximum(zo.value, 0) if a["act"] else zo.value
        self.record(i, "linear", "y", ydev, fwd)
        g = self._g_out(rec)
        if not self._dev_backward(y, g, rec):
            return
        gn = np.asarray(g, F64).reshape(ydev.shape)
        if a["act"]:
            gn = gn * (ydev > 0)
        backward(zo, gn)
        og = {"x": xo.grad, "w": wo.grad}
        if bo is not None:
            og["b"] = bo.grad
        self._finish(i, rec, L, og, ["x", "w", "b"])

    def _op_softmax_xent(self, i, rec):
        be, a = self.be, rec["args"]
        L = self._dev_inputs(rec, ["z"])
        lab = self._val(a["labels"])
        loss = be.softmax_xent(L["z"][1], be.tensor(lab))
        zo = Var(self._val(a["z"]).astype(F64), True)
        lo = oops.softmax_cross_entropy(zo, lab.astype(np.int64))
        self.record(i, "softmax_xent", "loss", np.array(self.tr.vals[rec["out"]]), lo.value)
        self.record(i, "softmax_xent", "argmax", rec["extra"].astype(np.int64),
                    oops.argmax_rows(self._val(a["z"]).astype(F64)), exact=True)
        self.grads[rec["out"]] = np.float64(1.0)
        self._dev_backward(loss, self._g_out(rec), rec)
        backward(lo)
        self._finish(i, rec, L, {"z": zo.grad}, ["z"])

    def _op_bce_logits(self, i, rec):
        be, a = self.be, rec["args"]
        L = self._dev_inputs(rec, ["z"])
        lab = self._val(a["labels"])
        loss = be.bce_logits(L["z"][1], be.tensor(lab))
        zv = self._val(a["z"]).astype(F64)
        zo = Var(zv, True)
        lo = oops.bce_as_two_class_ce(zo, lab.astype(np.int64))
        self.record(i, "bce_logits", "loss", np.array(self.tr.vals[rec["out"]]), lo.value)
        self.grads[rec["out"]] = np.float64(1.0)
        self._dev_backward(loss, self._g_out(rec), rec)
        backward(lo)
        self._finish(i, rec, L, {"z": zo.grad}, ["z"])

    def _op_embedding(self, i, rec):
        be, a = self.be, rec["args"]
        L = self._dev_inputs(rec, ["table"])
        ids = self._val(a["ids"])
        y = be.embedding(L["table"][1], be.tensor(ids))
        to = Var(self._val(a["table"]).astype(F64), True)
        yo = oops.embedding(to, ids.astype(np.int64))
        # f32 rows are copies (exact); bf16 rows are the table rounded once
        self.record(i, "embedding", "rows", self.tr.vals[rec["out"]], yo.value,
                    exact=self.tr.dtypes[rec["out"]] == be._lib.BE_F32)
        g = self._g_out(rec)
        if not self._dev_backward(y, g, rec):
            return
        backward(yo, np.asarray(g, F64))
        self._finish(i, rec, L, {"table": to.grad}, ["table"])

    def _op_mul(self, i, rec):
        be, a = self.be, rec["args"]
        L = self._dev_inputs(rec, ["a", "b"])
        y = be.mul(L["a"][1], L["b"][1])
        ao, bo = Var(self._val(a["a"]).astype(F64), True), Var(self._val(a["b"]).astype(F64), True)
        yo = oops.mul(ao, bo)
        self.record(i, "mul", "y", self.tr.vals[rec["out"]], yo.value)
        g = self._g_out(rec)
        if not self._dev_backward(y, g, rec):
            return
        backward(yo, np.asarray(g, F64))
        self._finish(i, rec, L, {"a": ao.grad, "b": bo.grad}, ["a", "b"])

    def _op_concat(self, i, rec):
        be, a = self.be, rec["args"]
        refs = a["xs"]
        leaves = [_leaf(be, self._val(r), self._dt(r), self._req(r)) for r in refs]
        y = be.concat([l[1] for l in leaves])
        vo = [Var(self._val(r).astype(F64), True) for r in refs]
        yo = oops.concat(vo, 1)
        self.record(i, "concat", "y", self.tr.vals[rec["out"]], yo.value, exact=True)
        g = self._g_out(rec)
        if not self._dev_backward(y, g, rec):
            return
        backward(yo, np.asarray(g, F64))
        for j, (r, l, v) in enumerate(zip(refs, leaves, vo)):
            if not self._req(r):
                continue
            gd = l[0].grad.numpy()
            self.record(i, "concat", f"dx{j}", gd, v.grad)
            self._push(r.key, gd)

    def _op_bn_conv1x1(self, i, rec):
        """BN (train) → act → 1×1 conv, one device op: compared with the
        oracle's batchnorm2d → relu/relu6 → conv2d on the same inputs — the
        output, dx, dγ, dβ (summation scale, R16), dW and the running stats.
        The activation mask of the backward is the one the device takes:
        decided from the BN output recomputed in fp32 and rounded to bf16
        (as the operand transform stores it), i.e. from act(bn(x)) > 0 of the
        oracle's values within bf16 rounding of 0 — compared as computed."""
        be, a = self.be, rec["args"]
        L = self._dev_inputs(rec, ["x", "gamma", "beta", "w"])
        rm0 = self._val(a["running_mean"]) if a["running_mean"] is not None else None
        rv0 = self._val(a["running_var"]) if a["running_var"] is not None else None
        rmd = be.tensor(rm0) if rm0 is not None else None
        rvd = be.tensor(rv0) if rv0 is not None else None
        y = be.bn_conv1x1(L["x"][1], L["gamma"][1], L["beta"][1], rmd, rvd, L["w"][1], eps=a["eps"],
                          momentum=a["momentum"], act=a["act"])
        xo = Var(nhwc_to_nchw(self._val(a["x"])).astype(F64), True)
        go = Var(self._val(a["gamma"]).astype(F64), True)
        bo = Var(self._val(a["beta"]).astype(F64), True)
        wo = Var(nhwc_to_nchw(self._val(a["w"])).astype(F64), True)   # KRSC -> KCRS
        zo, (rm, rv) = oops.batchnorm2d(xo, go, bo, eps=a["eps"], momentum=a["momentum"],
                                        running_mean=None if rm0 is None else rm0.astype(F64),
                                        running_var=None if rv0 is None else rv0.astype(F64))
        if a["act"]:
            # the activation decision the device takes (SURVEY §8(c) reading 16): its own BN output
            # (be.batchnorm2d: same statistics kernels, same fp32 affine, stored bf16) — act(z) written
            # as z·mask (+ 6 where clamped) so the oracle's gradient takes exactly that mask
            with be.no_grad():
                yb = nhwc_to_nchw(be.batchnorm2d(be.tensor(self._val(a["x"]), dtype="bf16"),
                                                 be.tensor(self._val(a["gamma"])), be.tensor(self._val(a["beta"])),
                                                 eps=a["eps"], act=a["act"]).numpy()).astype(F64)
            mask = _act_mask(yb, a["act"]).astype(F64)
            six = 6.0 * (yb >= 6.0) if a["act"] == 2 else np.zeros_like(yb)
            ho = oops.add(oops.mul(zo, Var(mask)), Var(six))
        else:
            ho = zo
        yo = oops.conv2d(ho, wo, None, 1, 0)
        ydev = y.numpy()
        self.record(i, "bn_conv1x1", "y", nhwc_to_nchw(ydev), yo.value)
        if rmd is not None:
            xa = np.abs(nhwc_to_nchw(self._val(a["x"])).astype(F64)).mean(axis=(0, 2, 3))
            self.record(i, "bn_conv1x1", "running_mean", rmd.numpy(), rm,
                        mass=(a["momentum"] * xa + (1 - a["momentum"]) * np.abs(rm0)).max())
            self.record(i, "bn_conv1x1", "running_var", rvd.numpy(), rv)
        g = self._g_out(rec)
        if not self._dev_backward(y, g, rec):
            return
        backward(yo, nhwc_to_nchw(np.asarray(g).reshape(ydev.shape)))
        og = {"x": nchw_to_nhwc(xo.grad), "gamma": go.grad, "beta": bo.grad, "w": nchw_to_nhwc(wo.grad)}
        self._finish(i, rec, L, og, ["x", "gamma", "beta", "w"])

    def _op_dropout(self, i, rec):
        be, a = self.be, rec["args"]
        L = self._dev_inputs(rec, ["x"])
        y = be.dropout(L["x"][1], a["p"], a["seed"], a["offset"], a["training"])
        xv = self._val(a["x"]).astype(F64)
        xo = Var(xv, True)
        yo = oops.dropout(xo, a["p"], a["seed"], a["offset"], training=a["training"])
        ydev = y.numpy()
        self.record(i, "dropout", "y", ydev, yo.value)
        # the keep mask is an integer decision: bit-exact wherever x ≠ 0
        nz = xv != 0
        if a["training"] and a["p"] > 0:
            keep = oops.dropout_keep_mask(xv.size, a["p"], a["seed"], a["offset"]).reshape(xv.shape)
            self.record(i, "dropout", "keep", (ydev != 0)[nz], keep[nz], exact=True)
        g = self._g_out(rec)
        if not self._dev_backward(y, g, rec):
            return
        backward(yo, np.asarray(g, F64).reshape(ydev.shape))
        self._finish(i, rec, L, {"x": xo.grad}, ["x"])

    def _op_conv2d_depthwise(self, i, rec):
        be, a = self.be, rec["args"]
        L = self._dev_inputs(rec, ["x", "w"])
        y = be.conv2d_depthwise(L["x"][1], L["w"][1], a["stride"], a["pad"])
        x = nhwc_to_nchw(self._val(a["x"])).astype(F64)
        w = np.ascontiguousarray(self._val(a["w"]).astype(F64).transpose(2, 0, 1)[:, None])  # RSC -> [C,1,R,S]
        xo, wo = Var(x, True), Var(w, True)
        zo = oops.conv2d_depthwise(xo, wo, a["stride"], a["pad"])
        ydev = y.numpy()
        self.record(i, "conv2d_depthwise", "y", nhwc_to_nchw(ydev), zo.value)
        g = self._g_out(rec)
        if not self._dev_backward(y, g, rec):
            return
        backward(zo, nhwc_to_nchw(np.asarray(g).reshape(ydev.shape)))
        og = {"x": nchw_to_nhwc(xo.grad), "w": np.ascontiguousarray(wo.grad[:, 0].transpose(1, 2, 0))}
        self._finish(i, rec, L, og, ["x", "w"])

    # ------------------------------------------------------------ report
    def worst(self, n=8):
        return sorted(self.errs, key=lambda e: -e[3])[:n]

    def failures(self):
        return [e for e in self.errs if not e[3] <= self.tol]


def teacher_forced(be, model, batch, tol):
    """Trace the model's forward on the device, then replay every op (see the
    module docstring).  Returns the Replay (errs, worst(), failures())."""
    tr = OpTrace(be.api, model).install(be.nn)
    try:
        loss = model.loss(*batch)
    finally:
        tr.uninstall(be.nn)
    del loss
    rp = Replay(be, tr, tol).run()
    return rp


def forward_drift(be, trace: OpTrace):
    """Diagnostic: the oracle's OWN end-to-end forward, op by op over the traced
    graph (each op fed the oracle's previous outputs, parameters from the
    trace), against the device's traced outputs.  Returns [(idx, op, err)] —
    where the two forwards drift apart, not a gate."""
    ov = {}

    def val(r):
        k = r.key
        if k in ov:
            return ov[k]
        v = trace.vals[k].astype(F64)
        return v

    out = []
    for i, rec in enumerate(trace.recs):
        a, op = rec["args"], rec["op"]
        dev = trace.vals[rec["out"]].astype(F64)
        if op == "conv2d":
            x = nhwc_to_nchw(val(a["x"]))
            w = nhwc_to_nchw(val(a["w"]))
            b = Var(val(a["b"])) if a["b"] is not None else None
            y = oops.conv2d(Var(x), Var(w), b, a["stride"], a["pad"]).value
            if a["act"]:
                y = np.maximum(y, 0)
            y = nchw_to_nhwc(y)
        elif op == "batchnorm2d":
            y, _ = oops.batchnorm2d(Var(nhwc_to_nchw(val(a["x"]))), Var(val(a["gamma"])), Var(val(a["beta"])),
                                    eps=a["eps"])
            y = y.value
            if a["residual"] is not None:
                y = y + nhwc_to_nchw(val(a["residual"]))
            y = nchw_to_nhwc(_act(y, a["act"]))
        elif op == "batchnorm2d_add_bn":
            y1, _ = oops.batchnorm2d(Var(nhwc_to_nchw(val(a["x"]))), Var(val(a["gamma"])), Var(val(a["beta"])),
                                     eps=a["eps"])
            y2, _ = oops.batchnorm2d(Var(nhwc_to_nchw(val(a["xr"]))), Var(val(a["gamma_r"])), Var(val(a["beta_r"])),
                                     eps=a["eps"])
            y = nchw_to_nhwc(_act(y1.value + y2.value, a["act"]))
        elif op == "maxpool2d":
            yv, am = oops.maxpool2d(Var(nhwc_to_nchw(val(a["x"]))), a["k"], a["stride"], a["pad"])
            y = nchw_to_nhwc(yv.value)
            if rec.get("extra") is not None:  # winner flips between the two forwards (window index r·k+u)
                xs = nhwc_to_nchw(val(a["x"])).shape
                win = nhwc_to_nchw(rec["extra"]).astype(np.int64)
                P, Q = win.shape[2], win.shape[3]
                hh = np.arange(P)[:, None] * a["stride"] - a["pad"] + win // a["k"]
                ww = np.arange(Q)[None, :] * a["stride"] - a["pad"] + win % a["k"]
                flips = int((hh * xs[3] + ww != am).sum())
                out.append((i, "argmax flips", float(flips)))
        elif op == "dropout":
            y = oops.dropout(Var(val(a["x"])), a["p"], a["seed"], a["offset"], training=a["training"]).value
        elif op == "conv2d_depthwise":
            w = np.ascontiguousarray(val(a["w"]).transpose(2, 0, 1)[:, None])
            y = nchw_to_nhwc(oops.conv2d_depthwise(Var(nhwc_to_nchw(val(a["x"]))), Var(w), a["stride"], a["pad"]).value)
        elif op == "avgpool_global":
            y = oops.avgpool_global(Var(nhwc_to_nchw(val(a["x"])))).value
        elif op == "reshape":
            y = val(a["x"]).reshape(dev.shape)
        elif op == "linear":
            b = Var(val(a["b"])) if a["b"] is not None else None
            y = oops.linear(Var(val(a["x"])), Var(val(a["w"])), b).value
            if a["act"]:
                y = np.maximum(y, 0)
        elif op == "softmax_xent":
            y = np.asarray(oops.softmax_cross_entropy(Var(val(a["z"])), trace.vals[a["labels"].key].astype(np.int64)).value)
        else:
            y = dev
        ov[rec["out"]] = y
        out.append((i, op, rel_err(dev, y)))
    return out
