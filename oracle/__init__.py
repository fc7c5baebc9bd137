"""ORACLE — plain, slow, obviously-correct float64 CPU implementation of the
eager training step (BASELINE.json north_star).  TEST INFRASTRUCTURE ONLY:
only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import it.  Shares no code with
paper_1912_01703_b200/ (the product path never imports this package).

Pins: tests/test_oracle_*.py check it against the paper's / SPEC's worked
values (tests/golden/), closed forms, brute force and finite differences.
"""
from . import autograd, ops, nets, optim, step, compare  # noqa: F401
