"""Conditioning floor of an end-to-end training step (test infrastructure).

The north_star tolerances (1e-4 fp32, 2e-2 bf16, ∞-norm per tensor) are met
op by op (tests/teacher.py).  End to end, a deep network at initialisation
can be so ill-conditioned that ANY implementation at a given arithmetic
resolution deviates from the float64 result by more than the tolerance: a
ReLU whose pre-activation lies within rounding distance of 0 flips its mask,
and the flipped unit's whole upstream gradient moves (SURVEY §8(c) readings
15-16).  This module measures that floor with the oracle alone: the relative
change (∞-norm, per tensor) of the oracle's own one-step gradients when every
parameter and every float input is perturbed by a relative ±u with random
signs, u = the arithmetic's unit roundoff: 2^-8 for bf16 operands, and
2^-21 for the fp32 path, whose GEMMs/convs are 3xTF32 (R10: with
hi = rna_tf32(x), lo = rna_tf32(x - hi), the dropped lo*lo' term and the
residuals x - hi - lo are each <= 2^-22 |x y|, so one product carries up to
~3 * 2^-22 ~= 2^-20.4 relative error, not fp32's 2^-24).  It is a
reported number, never a tolerance: the e2e tests gate, element-wise at the
north_star tolerance, exactly the tensors whose floor is at most half of it.
"""
from __future__ import annotations

import numpy as np

from oracle.compare import rel_err
from oracle.step import train_step

UNIT_ROUNDOFF = {"f32": 2.0 ** -21, "bf16": 2.0 ** -8}


def _perturb(a, u, rng):
    a = np.asarray(a)
    if not np.issubdtype(a.dtype, np.floating):
        return a
    return a.astype(np.float64) * (1.0 + u * rng.choice([-1.0, 1.0], size=a.shape))


def sensitivity(onet, params, batch, u, ref=None, draws=2, seed=0, lr=0.01):
    """{"loss": κ, "grad:<name>": κ, ...}: max over `draws` random-sign
    perturbations of the oracle's relative one-step change."""
    ref = ref if ref is not None else train_step(onet, params, batch, lr=lr)
    rng = np.random.default_rng(seed)
    kap = {}
    for _ in range(draws):
        P1 = {k: _perturb(v, u, rng) for k, v in params.items()}
        b1 = tuple(_perturb(a, u, rng) for a in batch)
        r1 = train_step(onet, P1, b1, lr=lr)
        cur = {"loss": rel_err(np.array(r1["loss"]), np.array(ref["loss"]))}
        for k in params:
            cur["grad:" + k] = rel_err(r1["grads"][k], ref["grads"][k])
        for k, v in cur.items():
            kap[k] = max(kap.get(k, 0.0), v)
    return kap
