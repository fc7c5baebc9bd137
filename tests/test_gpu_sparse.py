"""NCF sparse path on the B200 (-m gpu): embedding tables
registered with be_sgd_sparse are updated on their touched rows inside the
embedding backward (μ = 0, wd = 0; no gradient table), the dense tower with
momentum 0.9 / wd 1e-4 — compared with the float64 oracle's dense SGD on the
same step (oracle/optim.py; a zero gradient row leaves its row unchanged, so
the two are the same update).  Untouched rows must be bitwise unchanged."""
import numpy as np
import pytest

import synth
from gpu_common import be_init, rel
from oracle import nets as onets
from oracle.optim import sgd_step as oracle_sgd
from oracle.step import train_step

pytestmark = pytest.mark.gpu

TABLES = ("user_gmf", "item_gmf", "user_mlp", "item_mlp")


@pytest.mark.parametrize("overlap", [False, True])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_ncf_sparse_tables_one_step(dtype, overlap):
    be = be_init()
    be.set_compute_dtype(dtype)
    nu, ni, B = 500, 300, 2048  # many repeated ids per table
    onet = onets.NCF(n_users=nu, n_items=ni)
    pnet = be.nn.NCF(n_users=nu, n_items=ni)
    P = synth.make_params(onet.param_specs(), 51)
    users, items, y = synth.ncf_batch(B, nu, ni, 51)
    pnet.load(P)
    lr, mu, wd = 0.05, 0.9, 1e-4
    try:
        loss = be.nn.train_step(pnet, (be.tensor(users), be.tensor(items), be.tensor(y)), lr=lr, momentum=mu,
                                weight_decay=wd, overlap_sgd=overlap, sparse_embeddings=True)
        dev = {k: p.numpy() for k, p in pnet.params.items()}
        for t in TABLES:
            assert pnet.params[t].grad is None, "sparse tables carry no gradient tensor"
    finally:
        be.sgd_sparse([])
        be.sgd_overlap([])
    ref = train_step(onet, P, (users, items, y), lr=lr)  # gradients (the SGD below replaces its update)
    g = ref["grads"]
    tab_new, _ = oracle_sgd({k: P[k] for k in TABLES}, {k: g[k] for k in TABLES}, lr, 0.0, 0.0)
    dense = [k for k in P if k not in TABLES]
    den_new, _ = oracle_sgd({k: P[k] for k in dense}, {k: g[k] for k in dense}, lr, mu, wd)
    tol = 1e-4 if dtype == "f32" else 2e-2
    assert rel(np.array(loss.item()), np.array(ref["loss"])) <= tol
    for k, v in {**tab_new, **den_new}.items():
        assert rel(dev[k], v) <= tol, k
    # touched rows moved, untouched rows are bitwise unchanged
    for k, ids, n in (("user_gmf", users, nu), ("user_mlp", users, nu), ("item_gmf", items, ni),
                      ("item_mlp", items, ni)):
        untouched = np.setdiff1d(np.arange(n), ids)
        assert len(untouched) > 0
        assert np.array_equal(dev[k][untouched], P[k][untouched]), k
        assert not np.array_equal(dev[k][np.unique(ids)], P[k][np.unique(ids)]), k


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("B,V,D", [(8192, 138493, 64), (1000, 37, 128), (1, 5, 64), (12000, 26744, 128)])
def test_sparse_update_exact(B, V, D, dtype):
    """The touched-rows update in isolation, on exactly representable data:
    integer table values, upstream rows of small integers, lr = 2^-4 — every
    Σ g and every p − lr·Σ g is exact in fp32, so the device result must equal
    the oracle's SGD on the oracle's embedding gradient BITWISE (any dropped,
    duplicated or misrouted row contribution shows)."""
    from oracle import ops as oops
    from oracle.autograd import Var, backward
    be = be_init()
    be.set_compute_dtype(dtype)
    rng = np.random.default_rng(B + V + D)
    table = rng.integers(-50, 50, (V, D)).astype(np.float32)
    ids = rng.integers(0, V, B).astype(np.int32)
    g = rng.integers(-3, 4, (B, D)).astype(np.float32)
    lr = 2.0 ** -4
    t = be.tensor(table, requires_grad=True)
    be.sgd_sparse([t], lr)
    try:
        y = be.embedding(t, be.tensor(ids))
        y.backward(be.tensor(g, dtype="bf16" if dtype == "bf16" else None))
        got = t.numpy()
        assert t.grad is None
    finally:
        be.sgd_sparse([])
    to = Var(table.astype(np.float64), True)
    backward(oops.embedding(to, ids.astype(np.int64)), g.astype(np.float64))
    want, _ = oracle_sgd({"t": table}, {"t": to.grad}, lr)
    assert np.array_equal(got, want["t"].astype(np.float32))


def test_sparse_registration_errors():
    be = be_init()
    t = be.tensor(np.zeros((4, 8), np.float32), requires_grad=True)
    be.sgd_overlap([t], 0.1)
    try:
        with pytest.raises(be.BeError):
            be.sgd_sparse([t], 0.1)
    finally:
        be.sgd_overlap([])
    be.sgd_sparse([t], 0.1)
    try:
        with pytest.raises(be.BeError):
            be.sgd_step([t], 0.1)
    finally:
        be.sgd_sparse([])
