"""ORACLE — test infrastructure only.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import this package.
The product path (paper_1912_01703_b200/) never imports it.

Plain float64 reverse-mode tape (§4.3 "builds up a
representation of the computed function every time it is executed" /
"reverse-mode automatic differentiation, which computes the gradient of a
scalar output with respect to a multivariate input").

Contract followed:
  * every op executed with a recording input creates a Node holding its
    inputs and a vector-Jacobian-product closure;
  * backward(root) seeds d(root)=1 (scalar root), computes dependency counts
    over the reachable graph, runs nodes in reverse topological order, sums
    fan-out contributions, and accumulates (+=) into leaf .grad;
  * versions: each Var carries a version counter bumped by in-place writes;
    a node records the versions of the inputs its VJP reads and checks them
    at unpack (backward) time.
"""
from __future__ import annotations

import numpy as np

_grad_enabled = [True]


class VersionError(RuntimeError):
    pass


class Var:
    """A float64 (or int64) array plus tape metadata."""

    __slots__ = ("value", "grad", "node", "requires_grad", "version", "name")

    def __init__(self, value, requires_grad=False, name=""):
        self.value = np.asarray(value)
        self.grad = None
        self.node = None
        self.requires_grad = bool(requires_grad)
        self.version = 0
        self.name = name

    @property
    def is_leaf(self):
        return self.node is None

    def bump_version(self):
        self.version += 1


class Node:
    __slots__ = ("name", "inputs", "vjp", "saved_versions", "consumed")

    def __init__(self, name, inputs, vjp):
        self.name = name
        self.inputs = inputs
        self.vjp = vjp
        self.saved_versions = [v.version for v in inputs]
        self.consumed = False


class no_grad:
    def __enter__(self):
        self.prev = _grad_enabled[0]
        _grad_enabled[0] = False

    def __exit__(self, *a):
        _grad_enabled[0] = self.prev


def record(name, inputs, out_value, vjp):
    """Create the output Var of an op; attach a Node if any input records."""
    out = Var(out_value)
    if _grad_enabled[0] and any(v.requires_grad for v in inputs):
        out.requires_grad = True
        out.node = Node(name, list(inputs), vjp)
    return out


def backward(root: Var, upstream=None, retain_graph=False):
    """Reverse-mode sweep (S:320 dependency counts)."""
    if not root.requires_grad:
        raise RuntimeError("root does not require grad")
    if upstream is None:
        if root.value.size != 1:
            raise RuntimeError("MissingUpstreamForNonScalar")
        upstream = np.ones_like(root.value, dtype=np.float64)
    if root.node is None:  # root is a leaf
        root.grad = upstream.copy() if root.grad is None else root.grad + upstream
        return
    # 1. dependency counts over reachable nodes
    deps = {}
    stack = [root.node]
    seen = {id(root.node)}
    nodes = {id(root.node): root.node}
    while stack:
        n = stack.pop()
        if n.consumed:
            raise RuntimeError("DoubleBackwardWithoutRetain")
        for v in n.inputs:
            if v.node is not None:
                deps[id(v.node)] = deps.get(id(v.node), 0) + 1
                if id(v.node) not in seen:
                    seen.add(id(v.node))
                    nodes[id(v.node)] = v.node
                    stack.append(v.node)
    # 2. ready queue in reverse topological order
    pending = {id(root.node): np.asarray(upstream, dtype=np.float64)}
    ready = [root.node]
    while ready:
        n = ready.pop()
        g = pending.pop(id(n))
        for v, ver in zip(n.inputs, n.saved_versions):
            if v.version != ver:
                raise VersionError(f"VersionMismatch in {n.name}")
        grads = n.vjp(g)
        assert len(grads) == len(n.inputs), n.name
        if not retain_graph:
            n.consumed = True
        for v, gi in zip(n.inputs, grads):
            if gi is None or not v.requires_grad:
                pass
            elif v.node is None:  # leaf accumulate (+=)
                v.grad = np.array(gi, dtype=np.float64) if v.grad is None else v.grad + gi
            else:
                k = id(v.node)
                pending[k] = gi if k not in pending else pending[k] + gi
            if v.node is not None:
                k = id(v.node)
                deps[k] -= 1
                if deps[k] == 0:
                    if k not in pending:  # branch produced no gradient
                        pending[k] = np.zeros_like(v.value, dtype=np.float64)
                    ready.append(nodes[k])
