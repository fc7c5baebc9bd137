"""Runtime semantics on the B200 (-m gpu): caching allocator (PAPER.md:193-204
§5.3), immediate free, BE_SYNC bitwise
equivalence, bf16 end-to-end CNN parity (R8),
and the DDP code path through NCCL at world size 1."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import synth
from gpu_common import be_init, rel
from oracle import nets as onets, ops as oops
from oracle.step import train_step

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _fro(x, o):
    x, o = np.asarray(x, np.float64), np.asarray(o, np.float64)
    return float(np.linalg.norm(x - o) / max(np.linalg.norm(o), 1e-30))


def test_allocator_round_reuse_and_streams():
    be = be_init()
    import ctypes as C
    import torch
    call = be.api.call
    be.synchronize()
    be.empty_cache()  # start from an empty cache (other tests leave cached blocks)
    s0 = be.alloc_stats()
    p = C.c_uint64()
    call("be_raw_alloc", C.c_uint64(1000), C.c_uint64(0), C.byref(p))
    s1 = be.alloc_stats()
    assert s1["bytes_in_use"] - s0["bytes_in_use"] == 1024  # round_size(1000)
    call("be_raw_free", p)
    s2 = be.alloc_stats()
    assert s2["bytes_in_use"] == s0["bytes_in_use"] and s2["bytes_cached"] - s0["bytes_cached"] >= 1024
    # same size, same stream → cache hit, no raw allocation
    call("be_raw_alloc", C.c_uint64(1000), C.c_uint64(0), C.byref(p))
    s3 = be.alloc_stats()
    assert s3["cache_hit_count"] == s2["cache_hit_count"] + 1 and s3["raw_alloc_count"] == s2["raw_alloc_count"]
    call("be_raw_free", p)
    # another stream never reuses the first stream's pool
    other = torch.cuda.Stream()
    q = C.c_uint64()
    call("be_raw_alloc", C.c_uint64(1000), C.c_uint64(other.cuda_stream), C.byref(q))
    s4 = be.alloc_stats()
    assert s4["raw_alloc_count"] == s3["raw_alloc_count"] + 1
    call("be_raw_free", q)
    # double free is an error
    with pytest.raises(be.BeError) as e:
        call("be_raw_free", q)
    assert e.value.name in ("BE_E_DOUBLE_FREE", "BE_E_BAD_HANDLE")
    # conservation and empty_cache
    rel_bytes = be.empty_cache()
    s5 = be.alloc_stats()
    assert rel_bytes > 0 and s5["bytes_cached"] == 0
    assert be.empty_cache() == 0


def test_record_stream_defers_reuse():
    be = be_init()
    import torch
    be.synchronize()
    be.empty_cache()
    t = be.empty((1 << 18,), "f32")
    side = torch.cuda.Stream()
    be.api.call("be_record_stream", t.handle, __import__("ctypes").c_uint64(side.cuda_stream))
    with torch.cuda.stream(side):
        torch.cuda._sleep(20_000_000)  # keep the side stream busy
    s0 = be.alloc_stats()
    del t  # freed while still "in use" on the side stream → parked, not pooled
    u = be.empty((1 << 18,), "f32")
    s1 = be.alloc_stats()
    # the parked block is reused in STREAM ORDER: no new cudaMalloc, and the
    # compute stream now waits for the side stream's use before touching it
    assert s1["raw_alloc_count"] == s0["raw_alloc_count"]
    u.fill_(1.0)
    be.synchronize()                # the compute stream has drained...
    assert side.query()             # ...which it could only do after the side stream's work
    assert (u.numpy() == 1.0).all()
    del u


def test_immediate_free_flat_peak():
    """a create/drop loop keeps peak bytes flat (blocks return to
    the pool the moment their last reference dies)."""
    be = be_init()
    be.reset_peak()
    for _ in range(2000):
        a = be.empty((4096,), "f32")
        b = be.empty((4096,), "f32")
        del a, b
    s = be.alloc_stats()
    assert s["peak_bytes_in_use"] - s["bytes_in_use"] <= 2 * 16384


_SYNC_SCRIPT = r"""
import sys, json, numpy as np
sys.path.insert(0, {root!r})
import paper_1912_01703_b200 as be, synth
be.init(0)
be.set_compute_dtype("bf16")
net = be.nn.ResNet50(layers=(1, 1, 1, 1), base=16, classes=10)
net.load(synth.make_params(net.param_specs(), 0))
x = be.nn.images_to_device(synth.normal((4, 3, 64, 64), 0, 1), "bf16")
y = be.tensor(synth.labels(4, 10, 0))
for _ in range(2):
    be.nn.train_step(net, (x, y), lr=0.01, momentum=0.9)
h = __import__("hashlib").sha256()
for k, p in net.params.items():
    h.update(np.ascontiguousarray(p.numpy()).tobytes())
print(json.dumps({{"digest": h.hexdigest()}}))
"""


def _run_sync_script(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", _SYNC_SCRIPT.format(root=ROOT)], capture_output=True, text=True,
                       env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])["digest"]


def test_sync_mode_bitwise_equivalence():
    """BE_SYNC=1 (synchronise after every launch) gives bitwise the same
    parameters as the asynchronous run (acceptance #3), and two
    async runs agree bitwise (determinism: no floating-point atomics)."""
    a = _run_sync_script({"BE_SYNC": "0"})
    b = _run_sync_script({"BE_SYNC": "1"})
    c = _run_sync_script({"BE_SYNC": "0"})
    assert a == b == c


@pytest.mark.parametrize("C,act", [(64, 1), (64, 0), (256, 1), (24, 1)])
def test_bf16_bn_pool_residual_ops(C, act):
    """Per-op bf16 parity with identical (bf16-valued) inputs on both sides:
    BN(+ReLU) fwd/bwd, residual add+ReLU, 3×3/2 max pool (argmax included),
    global avg pool.  Outputs are single bf16 roundings of fp32 results →
    element-wise gate 1e-2 (bf16 has 8 significant bits)."""
    be = be_init()
    be.set_compute_dtype("bf16")
    from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
    from oracle.autograd import Var, backward
    q = lambda a: bf16_bits_to_f32(f32_to_bf16_bits(np.asarray(a, np.float32)))
    t = lambda a: np.ascontiguousarray(np.asarray(a).transpose(0, 2, 3, 1))
    tb = lambda a: np.ascontiguousarray(np.asarray(a).transpose(0, 3, 1, 2))
    rng = np.random.default_rng(C + act)
    N, H = 8, 14
    x = q(rng.standard_normal((N, C, H, H)) * 1.5 + 0.3)
    r = q(rng.standard_normal((N, C, H, H)))
    gam = (rng.standard_normal(C) * 0.3 + 1).astype(np.float32)
    bet = (rng.standard_normal(C) * 0.3).astype(np.float32)
    # oracle on the same values
    xo, ro = Var(x.astype(np.float64), True), Var(r.astype(np.float64), True)
    go, bo = Var(gam.astype(np.float64), True), Var(bet.astype(np.float64), True)
    yo, _ = oops.batchnorm2d(xo, go, bo)
    if act:
        yo = oops.relu(yo)
    # device
    xd, rd = be.tensor(t(x), requires_grad=True), be.tensor(t(r), requires_grad=True)
    gd, bd = be.tensor(gam, requires_grad=True), be.tensor(bet, requires_grad=True)
    yd = be.batchnorm2d(be.cast(xd, "bf16"), gd, bd, act=act)
    assert rel(tb(yd.numpy()), yo.value) < 1e-2
    # residual add + ReLU, then max pool and global average pool, fed the device's own y
    yv = tb(yd.numpy())
    zo = oops.relu(oops.add(Var(yv.astype(np.float64)), ro))
    zd = be.add_relu(yd, be.cast(rd, "bf16"))
    assert rel(tb(zd.numpy()), zo.value) < 1e-2
    zv = tb(zd.numpy())
    po, am = oops.maxpool2d(Var(zv.astype(np.float64)), 3, 2, 1)
    pd_, amd = be.maxpool2d(zd, 3, 2, 1, with_argmax=True)
    assert np.array_equal(tb(pd_.numpy()), po.value)  # max of stored values: exact
    win = tb(amd.numpy()).astype(np.int64)
    P = po.value.shape[2]
    hh = np.arange(P)[:, None] * 2 - 1 + win // 3
    ww = np.arange(P)[None, :] * 2 - 1 + win % 3
    assert np.array_equal(hh * H + ww, am)  # bit-exact winners on identical inputs
    ao = oops.avgpool_global(Var(tb(pd_.numpy()).astype(np.float64)))
    ad = be.avgpool_global(pd_)
    assert rel(ad.numpy(), ao.value) < 1e-2
    # backward through BN(+ReLU) with a bf16 upstream (mask from the device output)
    g = q(rng.standard_normal(yo.value.shape))
    backward(yo, g.astype(np.float64))
    yd2 = be.batchnorm2d(be.cast(xd, "bf16"), gd, bd, act=act)
    yd2.backward(be.tensor(t(g), dtype="bf16"))
    assert rel(tb(xd.grad.numpy()), xo.grad) < 2e-2
    assert rel(gd.grad.numpy(), go.grad) < 1e-2 and rel(bd.grad.numpy(), bo.grad) < 1e-2


def test_resnet_small_teacher_forced_bf16():
    """Every op of a small bf16 ResNet (all block types) fed the device's own
    inputs and upstream gradients vs the float64 oracle at 2e-2 element-wise
    (tests/teacher.py; the full-depth version is test_gpu_fulldepth.py)."""
    from teacher import teacher_forced
    be = be_init()
    be.set_compute_dtype("bf16")
    onet = onets.ResNet50(layers=(1, 1, 1, 1), base=16, classes=10)
    pnet = be.nn.ResNet50(layers=(1, 1, 1, 1), base=16, classes=10)
    pnet.load(synth.make_params(onet.param_specs(), 4))
    x = synth.bf16_values(synth.normal((8, 3, 64, 64), 4, 1))
    rp = teacher_forced(be, pnet, (be.nn.images_to_device(x, "bf16"), be.tensor(synth.labels(8, 10, 4))), 2e-2)
    print("worst:", rp.worst(4))
    assert not rp.failures(), rp.failures()[:8]


def test_ddp_world1_through_nccl_matches_single():
    """The DDP path (ncclBroadcast at attach, bucketed ncclAllReduce during
    backward on the comm stream, 1/world folded into SGD) at world size 1
    gives bitwise the same step as the plain path."""
    be = be_init()
    be.set_compute_dtype("bf16")
    import torch  # noqa: F401  (loads libnccl.so.2 for the library's dlopen)
    sizes = (256, 512, 256, 10)
    P = synth.make_params(onets.MLP(sizes).param_specs(), 5)
    x = be.tensor(synth.normal((64, 256), 5, 1), dtype="bf16")
    y = be.tensor(synth.labels(64, 10, 5))
    plain = be.nn.MLP(sizes).load(P)
    for _ in range(2):
        be.nn.train_step(plain, (x, y), lr=0.05, momentum=0.9)
    ddp = be.nn.MLP(sizes).load(P)
    try:
        be.dist_init(0, 1, be.dist_unique_id())
    except be.BeError as e:  # already initialised by another test in this process
        assert e.name == "BE_E_ARG"
    be.ddp_attach(ddp.parameters(), bucket_bytes=1 << 18)  # several buckets
    for _ in range(2):
        be.nn.train_step(ddp, (x, y), lr=0.05, momentum=0.9)
    be.synchronize()
    for k in P:
        assert np.array_equal(ddp.params[k].numpy(), plain.params[k].numpy()), k
    be.ddp_detach()
    # DDP + overlapped SGD: each bucket's params are updated on the comm stream
    # right behind its allreduce — still bitwise the plain step
    ddp2 = be.nn.MLP(sizes).load(P)
    be.ddp_attach(ddp2.parameters(), bucket_bytes=1 << 18)
    for _ in range(2):
        be.nn.train_step(ddp2, (x, y), lr=0.05, momentum=0.9, overlap_sgd=True)
    be.synchronize()
    for k in P:
        assert np.array_equal(ddp2.params[k].numpy(), plain.params[k].numpy()), k
    be.sgd_overlap([])
    be.ddp_detach()


def test_ddp_grad_accumulation_and_tied_weights():
    """DDP (world 1 through NCCL): gradients read right after backward are
    the reduced bucket values, two backward passes accumulate exactly as the
    plain path does (the bucket holds the mean, so re-reduction adds mean(g2)
    to mean(g1)), and a weight used twice in one graph (tied) is reduced only
    after both contributions landed."""
    be = be_init()
    be.set_compute_dtype("f32")
    import torch  # noqa: F401
    rng = np.random.default_rng(40)
    W0 = rng.standard_normal((64, 64)).astype(np.float32) / 8
    x1 = be.tensor(rng.standard_normal((16, 64)).astype(np.float32))
    x2 = be.tensor(rng.standard_normal((16, 64)).astype(np.float32))

    def run(W):
        for x in (x1, x2):  # tied: the same W applied twice, then a second backward accumulates
            be.sum(be.linear(be.linear(x, W), W)).backward()
        return W.grad.numpy()
    plain = run(be.tensor(W0, requires_grad=True))
    Wd = be.tensor(W0, requires_grad=True)
    try:
        be.dist_init(0, 1, be.dist_unique_id())
    except be.BeError as e:  # already initialised by an earlier test in this process
        assert e.name == "BE_E_ARG"
    assert be.dist_world() == (0, 1)
    be.ddp_attach([Wd], bucket_bytes=1 << 12)
    try:
        assert np.array_equal(run(Wd), plain)
        be.ddp_sync_buffers([be.tensor(np.ones(3, np.float32))])
    finally:
        be.ddp_detach()


@pytest.mark.parametrize("net", ["mlp", "resnet"])
def test_overlapped_sgd_bitwise_equals_fused(net):
    """be_sgd_overlap (each parameter updated inside backward, on a side
    stream, as soon as its gradient is final) gives bitwise the parameters of
    the fused be_sgd_step after several momentum steps — i.e. no update reads
    a partial gradient and no forward reads a stale parameter or bf16 shadow."""
    be = be_init()
    be.set_compute_dtype("bf16")
    from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
    if net == "mlp":
        sizes = (1024, 2048, 1536, 10)  # 2.1 M + 3.1 M params: several overlap groups
        P = synth.make_params(onets.MLP(sizes).param_specs(), 6)
        mk = lambda: be.nn.MLP(sizes).load(P)  # noqa: E731
        batch = (be.tensor(synth.normal((128, 1024), 6, 1), dtype="bf16"), be.tensor(synth.labels(128, 10, 6)))
    else:
        P = synth.make_params(onets.ResNet50(layers=(1, 1, 1, 1), base=16, classes=10).param_specs(), 6)
        mk = lambda: be.nn.ResNet50(layers=(1, 1, 1, 1), base=16, classes=10).load(P)  # noqa: E731
        x = bf16_bits_to_f32(f32_to_bf16_bits(synth.normal((8, 3, 64, 64), 6, 1)))
        batch = (be.nn.images_to_device(x, "bf16"), be.tensor(synth.labels(8, 10, 6)))
    # settle the per-shape kernel autotuner first (while it is still trying
    # candidates, two models stepping alternately would get different GEMM
    # variants — different, equally valid summation orders)
    scratch = mk()
    for _ in range(30):  # ≥ 4 calls per candidate (1 warm-up + 3 timed rounds)
        be.nn.train_step(scratch, batch, lr=0.05)
        be.nn.train_step(scratch, batch, lr=0.05, overlap_sgd=True)
    be.synchronize()
    for _ in range(2):
        be.nn.train_step(scratch, batch, lr=0.05)
    fused, over = mk(), mk()
    lf = lo = None
    for _ in range(3):
        lf = be.nn.train_step(fused, batch, lr=0.05, momentum=0.9, weight_decay=1e-4)
        lo = be.nn.train_step(over, batch, lr=0.05, momentum=0.9, weight_decay=1e-4, overlap_sgd=True)
    be.synchronize()
    assert lf.item() == lo.item()
    for k in P:
        assert np.array_equal(over.params[k].numpy(), fused.params[k].numpy()), k
    if net == "mlp":
        # the 2-D weights' updates ran inside their wgrad GEMM's epilogue
        # (fused SGD): no gradient tensor was ever materialised for them
        assert over.params["fc0.w"].grad is None and over.params["fc1.w"].grad is None
        assert over.params["fc0.b"].grad is not None
    # a registered parameter cannot also be stepped by be_sgd_step
    with pytest.raises(be.BeError) as ei:
        be.sgd_step(over.parameters(), 0.1)
    assert ei.value.name == "BE_E_ARG"
    be.sgd_overlap([])


@pytest.mark.parametrize("dt,C,act", [("bf16", 64, 1), ("bf16", 24, 0), ("f32", 40, 1), ("f32", 16, 0)])
def test_bn_fused_residual(dt, C, act):
    """batchnorm2d(..., residual=r): y = act(bn(x) + r) in one pass (the
    ResNet block output) vs the oracle's composition relu(add(bn(x), r)),
    forward and backward (dx, dγ, dβ and dr).  bf16: inputs bf16-valued on
    both sides, one rounding of the fp32 result → 1e-2; f32 → 1e-4."""
    be = be_init()
    be.set_compute_dtype(dt)
    from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
    from oracle.autograd import Var, backward
    q = (lambda a: bf16_bits_to_f32(f32_to_bf16_bits(np.asarray(a, np.float32)))) if dt == "bf16" else \
        (lambda a: np.asarray(a, np.float32))
    t = lambda a: np.ascontiguousarray(np.asarray(a).transpose(0, 2, 3, 1))
    tb = lambda a: np.ascontiguousarray(np.asarray(a).transpose(0, 3, 1, 2))
    tol = 1e-2 if dt == "bf16" else 1e-4
    rng = np.random.default_rng(C + act)
    N, H = 4, 9
    x = q(rng.standard_normal((N, C, H, H)) * 1.5 + 0.3)
    r = q(rng.standard_normal((N, C, H, H)))
    gam = (rng.standard_normal(C) * 0.3 + 1).astype(np.float32)
    bet = (rng.standard_normal(C) * 0.3).astype(np.float32)
    xo, ro = Var(x.astype(np.float64), True), Var(r.astype(np.float64), True)
    go, bo = Var(gam.astype(np.float64), True), Var(bet.astype(np.float64), True)
    yo, _ = oops.batchnorm2d(xo, go, bo)
    zo = oops.add(yo, ro)
    if act:
        zo = oops.relu(zo)
    xd, rd = be.tensor(t(x), requires_grad=True), be.tensor(t(r), requires_grad=True)
    gd, bd = be.tensor(gam, requires_grad=True), be.tensor(bet, requires_grad=True)
    xin = be.cast(xd, "bf16") if dt == "bf16" else xd
    rin = be.cast(rd, "bf16") if dt == "bf16" else rd
    calls0 = be.launch_count()
    zd = be.batchnorm2d(xin, gd, bd, act=act, residual=rin)
    assert rel(tb(zd.numpy()), zo.value) < tol
    g = q(rng.standard_normal(zo.value.shape))
    backward(zo, g.astype(np.float64))
    zd.backward(be.tensor(t(g), dtype=dt if dt == "bf16" else None))
    assert rel(tb(xd.grad.numpy()), xo.grad) < tol
    assert rel(tb(rd.grad.numpy()), ro.grad) < tol
    assert rel(gd.grad.numpy(), go.grad) < tol and rel(bd.grad.numpy(), bo.grad) < tol


@pytest.mark.parametrize("C,act,N,H", [(64, 1, 4, 9), (256, 1, 2, 14), (24, 0, 3, 7), (2048, 1, 2, 7)])
def test_bn_add_bn(C, act, N, H):
    """batchnorm2d_add_bn: act(bn(x) + bn_r(xr)) — the projection block output
    with the shortcut's BN applied in the same pass — vs the oracle's
    composition relu(add(bn(x), bn(xr))), forward (output and both BNs'
    running statistics) and backward (dx, dxr and the four affine gradients).
    bf16 inputs on both sides, fp32 arithmetic, one rounding → 1e-2."""
    be = be_init()
    be.set_compute_dtype("bf16")
    from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
    from oracle.autograd import Var, backward
    q = lambda a: bf16_bits_to_f32(f32_to_bf16_bits(np.asarray(a, np.float32)))
    t = lambda a: np.ascontiguousarray(np.asarray(a).transpose(0, 2, 3, 1))
    tb = lambda a: np.ascontiguousarray(np.asarray(a).transpose(0, 3, 1, 2))
    rng = np.random.default_rng(C + act + H)
    x = q(rng.standard_normal((N, C, H, H)) * 1.5 + 0.3)
    xr = q(rng.standard_normal((N, C, H, H)) * 0.7 - 0.2)
    p = [(rng.standard_normal(C) * 0.3 + 1).astype(np.float32), (rng.standard_normal(C) * 0.3).astype(np.float32),
         (rng.standard_normal(C) * 0.3 + 1).astype(np.float32), (rng.standard_normal(C) * 0.3).astype(np.float32)]
    rm0 = [(rng.standard_normal(C) * 0.1).astype(np.float32) for _ in range(2)]
    rv0 = [(rng.random(C) + 0.5).astype(np.float32) for _ in range(2)]
    xo, xro = Var(x.astype(np.float64), True), Var(xr.astype(np.float64), True)
    po = [Var(a.astype(np.float64), True) for a in p]
    y1, (rm1, rv1) = oops.batchnorm2d(xo, po[0], po[1], running_mean=rm0[0].astype(np.float64),
                                      running_var=rv0[0].astype(np.float64))
    y2, (rm2, rv2) = oops.batchnorm2d(xro, po[2], po[3], running_mean=rm0[1].astype(np.float64),
                                      running_var=rv0[1].astype(np.float64))
    zo = oops.add(y1, y2)
    if act:
        zo = oops.relu(zo)
    xd, xrd = be.tensor(t(x), requires_grad=True), be.tensor(t(xr), requires_grad=True)
    pd = [be.tensor(a, requires_grad=True) for a in p]
    rmd = [be.tensor(a) for a in rm0]
    rvd = [be.tensor(a) for a in rv0]
    zd = be.batchnorm2d_add_bn(be.cast(xd, "bf16"), pd[0], pd[1], rmd[0], rvd[0], be.cast(xrd, "bf16"), pd[2], pd[3],
                               rmd[1], rvd[1], act=act)
    assert rel(tb(zd.numpy()), zo.value) < 1e-2
    for dev, orc in ((rmd[0], rm1), (rvd[0], rv1), (rmd[1], rm2), (rvd[1], rv2)):
        assert rel(dev.numpy(), orc) < 1e-3
    g = q(rng.standard_normal(zo.value.shape))
    backward(zo, g.astype(np.float64))
    zd.backward(be.tensor(t(g), dtype="bf16"))
    assert rel(tb(xd.grad.numpy()), xo.grad) < 1e-2
    assert rel(tb(xrd.grad.numpy()), xro.grad) < 1e-2
    for dev, orc in zip(pd, po):
        assert rel(dev.grad.numpy(), orc.grad) < 1e-2


_TUNE_SCRIPT = r'''
import sys, json
sys.path[:0] = [{root!r}, {root!r} + "/tests"]
import numpy as np
import paper_1912_01703_b200 as be
be.init(0)
be.set_compute_dtype("bf16")
rng = np.random.default_rng(0)
x = be.tensor(rng.standard_normal((2, 14, 14, 256)).astype(np.float32), dtype="bf16")
w = be.tensor((rng.standard_normal((256, 3, 3, 256)) / 48).astype(np.float32), requires_grad=True)
g = be.tensor(rng.standard_normal((2, 14, 14, 256)).astype(np.float32), dtype="bf16")
outs = []
for _ in range(30):  # past every candidate's tuning rounds (≤ 5 variants × 4 rounds)
    be.zero_grad([w])
    y = be.conv2d(x, w, None, 1, 1)
    y.backward(g)
    outs.append(float(np.abs(w.grad.numpy()).sum()))
print(json.dumps({{"last": outs[-1]}}))
'''


def test_tune_file_replay(tmp_path):
    """BE_TUNE_FILE: a first process records its autotuning decisions, a second
    replays them without timing (no new lines) and computes the same result —
    the mechanism that keeps profiled runs on the unprofiled run's kernels."""
    tf = tmp_path / "tune.txt"
    env = dict(os.environ, BE_TUNE_FILE=str(tf))
    outs = []
    for _ in range(2):
        r = subprocess.run([sys.executable, "-c", _TUNE_SCRIPT.format(root=ROOT)], capture_output=True, text=True,
                           env=env, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1])["last"])
        if len(outs) == 1:
            first = tf.read_text().splitlines()
            assert first and all(len(line.split()) == 2 for line in first)
    assert tf.read_text().splitlines() == first  # the second run decided nothing new
    assert outs[0] == outs[1]
