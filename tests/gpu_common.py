"""Shared helpers for the -m gpu parity tests (test infrastructure)."""
import numpy as np
import pytest

_inited = [False]


def be_init():
    import paper_1912_01703_b200 as be
    if not _inited[0]:
        import torch
        if not torch.cuda.is_available():
            pytest.skip("needs a GPU")
        be.init(0)
        _inited[0] = True
    return be


def rel(x, o):
    from oracle.compare import rel_err
    return rel_err(x, o)


def run_product_step(be, model, specs_params, batch, lr=0.01, momentum=0.0, wd=0.0):
    """Load params, run one step on the device, return (loss, grads, new_params) in logical layout."""
    model.load(specs_params)
    params = model.parameters()
    be.zero_grad(params)
    loss = model.loss(*batch)
    loss.backward()
    grads = {n: model.logical(n, p.grad.numpy()) for n, p in model.params.items()}
    be.sgd_step(params, lr, momentum, wd)
    new = {n: model.logical(n, p.numpy()) for n, p in model.params.items()}
    return loss.item(), grads, new


def compare_step(oracle_out, loss, grads, new, tol, skip_zero_grad_names=()):
    errs = {"loss": rel(np.array(loss), np.array(oracle_out["loss"]))}
    for k, g in grads.items():
        errs["grad:" + k] = rel(g, oracle_out["grads"][k])
        errs["param:" + k] = rel(new[k], oracle_out["params"][k])
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, f"tolerance {tol} exceeded: {bad}"
    return errs


TOL = {"bf16": 2e-2, "f32": 1e-4}


def forward_error(be, pnet, dbatch):
    """The device forward's own deviation from exact arithmetic: the largest
    op-by-op drift of its traced forward against the oracle's forward over
    the same graph (tests/teacher.py forward_drift; every op of it is gated
    separately, teacher-forced)."""
    from teacher import OpTrace, forward_drift
    tr = OpTrace(be.api, pnet).install(be.nn)
    try:
        pnet.loss(*dbatch)
    finally:
        tr.uninstall(be.nn)
    d = [e for (_, op, e) in forward_drift(be, tr) if op != "argmax flips"]
    return max(d) if d else 0.0


def e2e_gate(be, onet, pnet, P, obatch, dbatch, dtype, verbose=True, name=""):
    """One SGD step on both sides vs the plain float64 oracle: every tensor's
    ∞-norm error reported beside the oracle's own conditioning floor κ
    (tests/conditioning.py), measured with a perturbation as large as the
    device forward's actual deviation (forward_error, at least the unit
    roundoff: in deep nets the forward drifts well above one rounding and
    flips near-tied max-pool winners / ReLU masks); gated at the north_star
    tolerance on the loss and on every gradient with κ ≤ tol/2 (a 0.8×-scaled
    gradient fails)."""
    from oracle.step import train_step
    from conditioning import UNIT_ROUNDOFF, sensitivity
    tol = TOL[dtype]
    ref = train_step(onet, P, obatch, lr=0.01)
    pnet.load(P)
    drift = forward_error(be, pnet, dbatch)
    loss, grads, new = run_product_step(be, pnet, P, dbatch)
    errs = {"loss": rel(np.array(loss), np.array(ref["loss"]))}
    for k in grads:
        errs["grad:" + k] = rel(grads[k], ref["grads"][k])
    u = max(UNIT_ROUNDOFF[dtype], drift)
    kappa = sensitivity(onet, P, obatch, u, ref=ref)
    gated = [k for k in errs if kappa[k] <= tol / 2]
    if verbose:
        print(f"{name} {dtype} e2e: loss err {errs['loss']:.2e}; {sum(errs[k] <= tol for k in errs)}/{len(errs)} "
              f"tensors ≤ {tol}; forward drift {drift:.2e} → κ at u = {u:.2e}; gated {len(gated)}")
        for k in sorted(errs, key=lambda k: -errs[k])[:8]:
            print(f"   {k:24s} err {errs[k]:.2e}   κ {kappa[k]:.2e}")
    assert errs["loss"] <= tol, errs["loss"]
    bad = {k: (errs[k], kappa[k]) for k in gated if not errs[k] <= tol}
    assert not bad, bad
    return errs, kappa
