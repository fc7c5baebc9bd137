"""ORACLE — test infrastructure only (see oracle/autograd.py header).

Parity comparator (reading 14): per tensor
    err = max_i |x_i − o_i| / max(max_i |o_i|, 1e-30)
(∞-norm relative error).  If max|o| == 0 the candidate must be exactly 0.
Gates: 1e-4 (fp32 / 3xTF32 path), 2e-2 (bf16 path) — BASELINE.json
north_star.  Integer tensors compare with ==.
"""
from __future__ import annotations

import numpy as np

TOL = {"f32": 1e-4, "bf16": 2e-2}


def rel_err(x, o) -> float:
    x = np.asarray(x, np.float64)
    o = np.asarray(o, np.float64)
    assert x.shape == o.shape, (x.shape, o.shape)
    if x.size == 0:
        return 0.0
    den = np.max(np.abs(o))
    if den == 0:
        return 0.0 if np.max(np.abs(x)) == 0 else float("inf")
    return float(np.max(np.abs(x - o)) / max(den, 1e-30))


def check(name, x, o, tol):
    e = rel_err(x, o)
    assert e <= tol, f"{name}: max rel err {e:.3e} > {tol:.1e}"
    return e
