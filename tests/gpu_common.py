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
