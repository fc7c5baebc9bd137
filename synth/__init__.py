"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic: it only draws numbers.
Both sides of every parity test take their inputs (weights, images, labels,
ids) from here as identical float32 / int32 host bytes, so no RNG-parity
question arises (SURVEY.md §8(c) reading 5).

Recipe (SURVEY.md §8(d) "Synthetic inputs"):
  * generator: NumPy Philox keyed by (seed, stream) — counter based, stable
    across platforms and NumPy versions;
  * weights: W ~ N(0,1)/sqrt(fan_in), b ~ N(0,1)/sqrt(fan_in) (SPEC S:614
    reading of Listing 1's unscaled randn); BN gamma=1,
    beta=0;
  * CNN images N(0,1); MLP-784 inputs U[0,1) (pixel-like); MLP-4096 inputs
    N(0,1); labels uniform in [0, classes); NCF ids uniform, label 1 w.p. 0.2.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "generator", "normal", "uniform", "labels", "make_params", "ncf_batch", "bf16_values",
]


def generator(seed: int, stream: int) -> np.random.Generator:
    """Counter-based generator for (seed, stream)."""
    return np.random.Generator(np.random.Philox(key=[int(seed) & (2**64 - 1),
                                                     int(stream) & (2**64 - 1)]))


def normal(shape, seed: int, stream: int) -> np.ndarray:
    return generator(seed, stream).standard_normal(size=tuple(shape),
                                                   dtype=np.float64).astype(np.float32)


def uniform(shape, seed: int, stream: int) -> np.ndarray:
    return generator(seed, stream).random(size=tuple(shape)).astype(np.float32)


def labels(n: int, classes: int, seed: int, stream: int = 7) -> np.ndarray:
    return generator(seed, stream).integers(0, classes, size=(n,), dtype=np.int64).astype(np.int32)


def make_params(specs, seed: int) -> dict:
    """specs: list of (name, shape, init, fan_in) with init in
    {"normal", "ones", "zeros"}.  Returns {name: float32 array}.

    Stream ids are 1000 + position so parameter draws never collide with
    input draws (streams < 1000)."""
    out = {}
    for i, (name, shape, init, fan_in) in enumerate(specs):
        if init == "normal":
            v = normal(shape, seed, 1000 + i).astype(np.float64) / np.sqrt(float(fan_in))
            out[name] = v.astype(np.float32)
        elif init == "ones":
            out[name] = np.ones(shape, np.float32)
        elif init == "zeros":
            out[name] = np.zeros(shape, np.float32)
        else:
            raise ValueError(init)
    return out


def ncf_batch(batch: int, n_users: int, n_items: int, seed: int):
    g = generator(seed, 11)
    users = g.integers(0, n_users, size=(batch,), dtype=np.int64).astype(np.int32)
    items = g.integers(0, n_items, size=(batch,), dtype=np.int64).astype(np.int32)
    y = (g.random(size=(batch,)) < 0.2).astype(np.int32)
    return users, items, y


def bf16_values(a) -> np.ndarray:
    """The bf16 configs' inputs are bfloat16 numbers (BASELINE configs C2-C5:
    "bf16"): round a draw to the nearest bfloat16 (RN-even on the float32
    bits; NaN/inf pass through) and return it as float32.  Data generation
    only — both sides receive these identical values."""
    x = np.ascontiguousarray(np.asarray(a, dtype=np.float64).astype(np.float32))
    bits = x.view(np.uint32).astype(np.uint64)
    rounded = ((bits + 0x7FFF + ((bits >> 16) & 1)) >> 16) << 16
    out = rounded.astype(np.uint32).view(np.float32)
    return np.where(np.isfinite(x), out, x).astype(np.float32)
