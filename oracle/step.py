"""ORACLE — test infrastructure only (see oracle/autograd.py header).

One eager training step = forward operator stream, reverse-mode tape to
gradients, SGD update (BASELINE.json north_star; §5.2,
PAPER.md:158-159 §4.3), optionally emulating R data-parallel replicas
(§5.4 "synchronize gradients using all-reduce style
primitives"):
  * the global batch is sharded contiguously, rank r gets rows
    [r·B/R, (r+1)·B/R);
  * each shard runs forward + backward on its own (BN statistics local);
  * g = (1/R) Σ_r g_r, then one SGD step; all replicas hold the same params.
"""
from __future__ import annotations

import numpy as np

from .autograd import Var, backward
from .optim import sgd_step


def _shard(batch, r, R):
    out = []
    for a in batch:
        B = a.shape[0]
        assert B % R == 0
        s = B // R
        out.append(a[r * s:(r + 1) * s])
    return tuple(out)


def train_step(net, params: dict, batch, lr=0.01, momentum=0.0, weight_decay=0.0,
               replicas=1, bufs=None):
    """params: {name: float32/float64 array}.  Returns dict with
    loss (mean over replicas), grads (averaged), params (updated), bufs,
    extras (per-replica forward extras)."""
    grads_sum = {k: np.zeros(np.shape(v), np.float64) for k, v in params.items()}
    losses, extras = [], []
    for r in range(replicas):
        P = {k: Var(np.asarray(v, np.float64), requires_grad=True, name=k)
             for k, v in params.items()}
        loss, ex = net.loss(P, _shard(batch, r, replicas))
        backward(loss)
        losses.append(float(loss.value))
        extras.append(ex)
        for k, v in P.items():
            if v.grad is not None:
                grads_sum[k] += v.grad
    grads = {k: g / replicas for k, g in grads_sum.items()}
    new_params, new_bufs = sgd_step(params, grads, lr, momentum, weight_decay, bufs)
    return {"loss": float(np.mean(losses)), "grads": grads, "params": new_params,
            "bufs": new_bufs, "extras": extras}
