"""One-step parity of the MLP training step (C1 fp32/3xTF32 at 1e-4; C2 bf16
at 2e-2) through the C ABI against the float64 oracle (-m gpu)."""
import numpy as np
import pytest

import synth
from gpu_common import be_init, run_product_step, compare_step, rel
from oracle import nets as onets
from oracle.step import train_step

pytestmark = pytest.mark.gpu


def _mlp_case(sizes, B, dtype, seed, uniform):
    be = be_init()
    be.set_compute_dtype(dtype)
    onet = onets.MLP(sizes)
    pnet = be.nn.MLP(sizes)
    assert onet.param_specs() == pnet.param_specs()
    P = synth.make_params(onet.param_specs(), seed)
    x = (synth.uniform if uniform else synth.normal)((B, sizes[0]), seed, 1)
    y = synth.labels(B, sizes[-1], seed)
    if dtype == "bf16":  # the bf16 configs' inputs are bf16 numbers; both sides get the same values
        x = synth.bf16_values(x)
    ref = train_step(onet, P, (x, y), lr=0.01)  # plain float64 oracle
    loss, grads, new = run_product_step(be, pnet, P, (be.tensor(x, dtype=dtype), be.tensor(y)))
    return ref, loss, grads, new


def test_c1_mlp_fp32_one_step():
    """C1: MLP 784-128-10, batch 64, fp32 (3xTF32 GEMMs), one SGD step."""
    ref, loss, grads, new = _mlp_case((784, 128, 10), 64, "f32", 0, True)
    errs = compare_step(ref, loss, grads, new, 1e-4)
    print("C1 max err", max(errs.values()))


@pytest.mark.parametrize("B", [1, 37, 300])
def test_mlp_fp32_ragged_batches(B):
    ref, loss, grads, new = _mlp_case((96, 136, 24), B, "f32", B, False)
    compare_step(ref, loss, grads, new, 1e-4)


def test_mlp_bf16_small():
    """bf16 MLP (ragged sizes, B = 200): every op teacher-forced at 2e-2, and
    one end-to-end step against the plain float64 oracle gated on the loss and
    on every well-conditioned gradient (gpu_common.e2e_gate)."""
    from teacher import teacher_forced
    from gpu_common import e2e_gate
    be = be_init()
    be.set_compute_dtype("bf16")
    sizes, B = (256, 512, 384, 100), 200
    onet, pnet = onets.MLP(sizes), be.nn.MLP(sizes)
    P = synth.make_params(onet.param_specs(), 1)
    x = synth.bf16_values(synth.normal((B, sizes[0]), 1, 1))
    y = synth.labels(B, sizes[-1], 1)
    pnet.load(P)
    rp = teacher_forced(be, pnet, (be.tensor(x, dtype="bf16"), be.tensor(y)), 2e-2)
    assert not rp.failures(), rp.failures()
    e2e_gate(be, onet, pnet, P, (x, y), (be.tensor(x, dtype="bf16"), be.tensor(y)), "bf16", name="mlp-small")


def test_loss_backward_accumulates_and_zero_grad_releases():
    be = be_init()
    be.set_compute_dtype("f32")
    x = be.tensor(np.array([1.0, 2.0, 3.0], np.float32), requires_grad=True)
    for _ in range(2):
        be.sum(be.mul(x, x)).backward()
    assert np.array_equal(x.grad.numpy(), np.array([4.0, 8.0, 12.0], np.float32))  # S:266 twice
    before = be.alloc_stats()["bytes_in_use"]
    be.zero_grad([x])
    assert x.grad is None
    assert be.alloc_stats()["bytes_in_use"] < before


def test_version_error_and_double_backward():
    be = be_init()
    be.set_compute_dtype("f32")
    w = be.tensor(np.ones(4, np.float32), requires_grad=True)
    a = be.tensor(np.arange(4, dtype=np.float32))
    y = be.sum(be.mul(w, a))
    a.fill_(2.0)  # mutate a saved input
    with pytest.raises(be.BeError) as e:
        y.backward()
    assert e.value.name == "BE_E_VERSION"
    y2 = be.sum(be.mul(w, w))
    y2.backward()
    with pytest.raises(be.BeError) as e:
        y2.backward()
    assert e.value.name == "BE_E_DOUBLE_BACKWARD"


def test_allocator_warmup_then_no_raw_allocs():
    """PAPER.md:249 (Fig. 2): iteration 1 pays cudaMalloc; later iterations
    reuse the per-stream cache."""
    be = be_init()
    be.set_compute_dtype("bf16")
    net = be.nn.MLP((512, 512, 10))
    P = synth.make_params(net.param_specs(), 0)
    net.load(P)
    x = be.tensor(synth.normal((128, 512), 0, 1), dtype="bf16")
    y = be.tensor(synth.labels(128, 10, 0))
    be.nn.train_step(net, (x, y))
    be.synchronize()
    s1 = be.alloc_stats()
    for _ in range(3):
        be.nn.train_step(net, (x, y))
    be.synchronize()
    s2 = be.alloc_stats()
    assert s2["raw_alloc_count"] == s1["raw_alloc_count"]
    assert s2["cache_hit_count"] > s1["cache_hit_count"]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_softmax_xent_argmax_bit_exact(dtype):
    """The softmax-CE kernel's argmax output (first maximum per row, SURVEY
    §8(c)-9 / reading 7) equals the oracle's bit-exactly on identical logits,
    including exact ties (rows repeating their max) and C not a multiple of
    the kernel's vector width; loss and dz at the dtype's tolerance."""
    from oracle import ops as oops
    from oracle.autograd import Var, backward
    be = be_init()
    B, Cc = 300, 1000
    z = synth.normal((B, Cc), 41, 1) * 3
    z[::7, 5] = z[::7].max(1) + 1.0
    z[::7, 900] = z[::7, 5]          # tie: first index (5) must win
    z[1::11, :] = 0.0                # all-equal rows → index 0
    z = synth.bf16_values(z) if dtype == "bf16" else z
    y = synth.labels(B, Cc, 41)
    zd = be.tensor(z, requires_grad=dtype == "f32", dtype=dtype)
    loss, am = be.softmax_xent(zd, be.tensor(y), with_argmax=True)
    assert np.array_equal(am.numpy().astype(np.int64), oops.argmax_rows(z.astype(np.float64)))
    zo = Var(z.astype(np.float64), True)
    lo = oops.softmax_cross_entropy(zo, y)
    backward(lo)
    assert rel(np.array(loss.item()), lo.value) < (1e-5 if dtype == "f32" else 2e-2)
