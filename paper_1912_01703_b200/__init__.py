"""paper_1912_01703_b200 — a B200-native (sm_100a) implementation of the
eager, define-by-run training step of arXiv 1912.01703 (PyTorch): forward
operator stream, reverse-mode tape, fused SGD, caching allocator, bucketed
NCCL gradient allreduce.  All compute runs in libbe.so (see include/be.h);
this package is the argument-marshalling layer plus the model programs.
"""
from .api import *  # noqa: F401,F403
from .api import Tensor, init, tensor, empty, no_grad  # noqa: F401
from . import nn  # noqa: F401
from ._lib import BeError, LIB_PATH  # noqa: F401
