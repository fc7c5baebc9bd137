"""ORACLE — test infrastructure only (see oracle/autograd.py header).

SGD (the paper names optimizers without formulas):
    p ← p − lr·(g + wd·p)
with momentum μ (PyTorch convention):
    g' = g + wd·p;  v₁ = g';  v ← μ·v + g';  p ← p − lr·v.
"""
from __future__ import annotations

import numpy as np


def sgd_step(params: dict, grads: dict, lr: float, momentum: float = 0.0,
             weight_decay: float = 0.0, bufs: dict | None = None):
    """Returns (new_params, new_bufs); inputs are not modified."""
    new_p, new_b = {}, {}
    for k, p in params.items():
        p = np.asarray(p, dtype=np.float64)
        if k not in grads or grads[k] is None:
            raise RuntimeError(f"MissingGradient: {k}")
        g = np.asarray(grads[k], dtype=np.float64) + weight_decay * p
        if momentum != 0.0:
            v = g if (bufs is None or k not in bufs) else momentum * bufs[k] + g
            new_b[k] = v
            g = v
        new_p[k] = p - lr * g
    return new_p, new_b
