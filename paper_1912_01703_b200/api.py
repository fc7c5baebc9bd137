"""Python face of the library: a Tensor handle class and one function per
be_op (argument marshalling only — the ops run in libbe.so on the GPU).

Mirrors the user-visible API of the paper's Listing 1/2:
tensors, differentiable ops, `loss.backward()`, an SGD step.
"""
from __future__ import annotations

import contextlib
import ctypes as C

import numpy as np

from . import _lib as L
from ._lib import call

_NP = {L.BE_F32: np.float32, L.BE_F64: np.float64, L.BE_I64: np.int64, L.BE_BOOL: np.bool_,
       L.BE_I32: np.int32, L.BE_U8: np.uint8, L.BE_BF16: np.uint16}
_FROM_NP = {np.dtype(np.float32): L.BE_F32, np.dtype(np.float64): L.BE_F64, np.dtype(np.int64): L.BE_I64,
            np.dtype(np.bool_): L.BE_BOOL, np.dtype(np.int32): L.BE_I32, np.dtype(np.uint8): L.BE_U8}
DTYPES = {"f32": L.BE_F32, "bf16": L.BE_BF16, "i32": L.BE_I32, "i64": L.BE_I64, "u8": L.BE_U8, "f64": L.BE_F64}


def _dt(d):
    if isinstance(d, str):
        return DTYPES[d]
    return int(d)


def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Host-side RN-even fp32 → bf16 bit pattern (input marshalling only)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u >> 16) & 1) + 0x7FFF
    return ((u + r) >> 16).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32)


class Tensor:
    """Owns one reference to a be_tensor handle (released in __del__)."""
    __slots__ = ("_h", "__weakref__")

    def __init__(self, handle):
        if not handle:
            raise ValueError("null tensor handle")
        self._h = C.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        try:
            if h is not None and h.value and L._lib is not None:
                L._lib.be_release(h)
                self._h = None
        except (AttributeError, TypeError):  # interpreter shutdown: module globals already cleared
            pass

    @property
    def handle(self):
        return self._h

    def _info(self):
        r = C.c_int()
        shp = (C.c_int64 * 6)()
        strd = (C.c_int64 * 6)()
        dt = C.c_int()
        ptr = C.c_uint64()
        call("be_tensor_info", self._h, C.byref(r), shp, strd, C.byref(dt), C.byref(ptr))
        return r.value, tuple(shp[:r.value]), tuple(strd[:r.value]), dt.value, ptr.value

    @property
    def shape(self):
        return self._info()[1]

    @property
    def dtype(self):
        return self._info()[3]

    @property
    def data_ptr(self):
        return self._info()[4]

    @property
    def version(self):
        v = C.c_uint64()
        call("be_tensor_version", self._h, C.byref(v))
        return v.value

    @property
    def requires_grad(self):
        v = C.c_int()
        call("be_tensor_requires_grad", self._h, C.byref(v))
        return bool(v.value)

    @property
    def grad(self):
        out = C.c_void_p()
        call("be_grad", self._h, C.byref(out))
        return Tensor(out.value) if out.value else None

    def numel(self):
        return int(np.prod(self.shape)) if self.shape else 1

    def numpy(self) -> np.ndarray:
        """Synchronous copy to host; bf16 is returned widened to float32."""
        rank, shape, _, dt, _ = self._info()
        out = np.empty(shape, dtype=_NP[dt])
        call("be_tensor_to_host", self._h, out.ctypes.data_as(C.c_void_p), C.c_size_t(out.nbytes))
        if dt == L.BE_BF16:
            return bf16_bits_to_f32(out)
        return out

    def item(self) -> float:
        v = C.c_double()
        call("be_item", self._h, C.byref(v))
        return v.value

    def backward(self, upstream: "Tensor | None" = None, retain_graph=False):
        call("be_backward", self._h, upstream._h if upstream is not None else None, int(retain_graph))

    def detach(self):
        out = C.c_void_p()
        call("be_detach", self._h, C.byref(out))
        return Tensor(out.value)

    def fill_(self, v):
        call("be_fill_", self._h, C.c_double(v))
        return self

    def copy_(self, src: "Tensor"):
        call("be_copy_", self._h, src._h)
        return self

    def __repr__(self):
        return f"be.Tensor(shape={self.shape}, dtype={self.dtype})"


# ------------------------------------------------------------------ construction
def init(device: int = 0, stream: int = 0):
    """Bind to a CUDA device; `stream` = cudaStream_t as int (e.g. torch's
    current stream `.cuda_stream`) or 0 for an own stream."""
    call("be_init", int(device), C.c_uint64(int(stream)))


def get_stream() -> int:
    v = C.c_uint64()
    call("be_get_stream", C.byref(v))
    return v.value


def launch_count() -> int:
    v = C.c_uint64()
    call("be_launch_count", C.byref(v))
    return v.value


def tensor(a, requires_grad=False, dtype=None) -> Tensor:
    """Create from host data (host→device copy on the compute stream).
    dtype "bf16" converts float32 host data with RN-even."""
    a = np.asarray(a)
    if dtype is not None and _dt(dtype) == L.BE_BF16:
        host = f32_to_bf16_bits(a.astype(np.float32))
        dt = L.BE_BF16
    else:
        if dtype is not None:
            a = a.astype(_NP[_dt(dtype)])
        elif a.dtype == np.float64:
            a = a.astype(np.float32)
        elif a.dtype == np.int64:
            a = a.astype(np.int32)
        host = np.ascontiguousarray(a)
        dt = _FROM_NP[host.dtype]
    shape = (C.c_int64 * 6)(*host.shape)
    out = C.c_void_p()
    call("be_tensor_create", host.ctypes.data_as(C.c_void_p), shape, host.ndim, dt, int(requires_grad),
         C.byref(out))
    call("be_synchronize")  # host buffer may be pageable / temporary
    return Tensor(out.value)


def empty(shape, dtype="f32") -> Tensor:
    shp = (C.c_int64 * 6)(*shape)
    out = C.c_void_p()
    call("be_tensor_empty", shp, len(shape), _dt(dtype), C.byref(out))
    return Tensor(out.value)


_KEEP = {}


def from_device(ptr: int, shape, dtype="f32", owner=None) -> Tensor:
    """Zero-copy wrap of device memory; `owner` is kept alive until release
    (PAPER.md:140-143)."""
    shp = (C.c_int64 * 6)(*shape)
    key = C.c_void_p(id(owner) if owner is not None else 0)

    def _release(ctx):
        _KEEP.pop(ctx, None)
    cb = L.RELEASE_CB(_release)
    out = C.c_void_p()
    call("be_tensor_from_device", C.c_void_p(ptr), shp, None, len(shape), _dt(dtype), cb, key, C.byref(out))
    _KEEP[key.value] = (owner, cb)
    return Tensor(out.value)


def from_torch(t) -> Tensor:
    """Zero-copy view of a contiguous CUDA torch tensor (plumbing only)."""
    import torch
    m = {torch.float32: "f32", torch.bfloat16: "bf16", torch.int32: "i32", torch.int64: "i64", torch.uint8: "u8"}
    assert t.is_cuda and t.is_contiguous()
    return from_device(t.data_ptr(), tuple(t.shape), m[t.dtype], owner=t)


# ------------------------------------------------------------------ ops
def _op(op, ins, attrs=None, n_out=1):
    arr = (C.c_void_p * len(ins))(*[t._h.value if t is not None else None for t in ins])
    outs = (C.c_void_p * n_out)()
    call("be_op", L.OPS[op], arr, len(ins), C.byref(attrs) if attrs is not None else None, outs, n_out)
    res = [Tensor(o) if o else None for o in outs]
    return res[0] if n_out == 1 else tuple(res)


def linear(x, w, b=None, act=0, out_f32=False):
    return _op("LINEAR", [x, w] + ([b] if b is not None else []), L.be_linear_attrs(int(act), int(out_f32)))


def matmul(a, b):
    return _op("MATMUL", [a, b])


def add(a, b, relu=False):
    return _op("ADD", [a, b], C.c_int(1 if relu else 0))


def add_relu(a, b):
    return _op("ADD_RELU", [a, b])


def mul(a, b):
    return _op("MUL", [a, b])


def relu(x):
    return _op("RELU", [x])


def softmax_xent(z, labels, with_argmax=False):
    return _op("SOFTMAX_XENT", [z, labels], None, 2 if with_argmax else 1)


def bce_logits(z, labels):
    return _op("BCE_LOGITS", [z, labels])


def conv2d(x, w, b=None, stride=1, pad=0, act=0, out_f32=False, bn_stats=False):
    """bn_stats=True: the output feeds batchnorm2d — its statistics come from
    the conv's epilogue (be_conv_attrs.bn_stats)."""
    return _op("CONV2D", [x, w] + ([b] if b is not None else []),
               L.be_conv_attrs(int(stride), int(pad), int(act), int(out_f32), int(bn_stats)))


def conv2d_depthwise(x, w, stride=1, pad=1):
    """Depthwise 3×3 convolution: x NHWC (C % 8 == 0), w f32 RSC [3, 3, C]."""
    return _op("CONV2D_DEPTHWISE", [x, w], L.be_dwconv_attrs(int(stride), int(pad)))


def dropout(x, p, seed, offset=0, training=True):
    """Inverted dropout with the counter-based Philox mask of (seed, offset)
    (include/be.h BE_OP_DROPOUT): the backward pass regenerates it."""
    return _op("DROPOUT", [x], L.be_dropout_attrs(float(p), int(bool(training)), int(seed) & (2**64 - 1),
                                                   int(offset) & (2**64 - 1)))


def maxpool2d(x, k=3, stride=2, pad=0, with_argmax=False):
    return _op("MAXPOOL2D", [x], L.be_pool_attrs(k, stride, pad), 2 if with_argmax else 1)


def avgpool_global(x):
    return _op("AVGPOOL_GLOBAL", [x])


def batchnorm2d(x, gamma, beta, running_mean=None, running_var=None, eps=1e-5, momentum=0.1, act=0, residual=None):
    """Train-mode batch norm; `residual` fuses the ResNet block output
    act(bn(x) + residual) into the same pass."""
    ins = [x, gamma, beta]
    if running_mean is not None:
        ins += [running_mean, running_var]
    if residual is not None:
        ins += [residual]
    return _op("BATCHNORM2D", ins, L.be_bn_attrs(eps, momentum, int(act), int(residual is not None)))


def batchnorm2d_add_bn(x, gamma, beta, running_mean, running_var, xr, gamma_r, beta_r, running_mean_r,
                       running_var_r, eps=1e-5, momentum=0.1, act=1):
    """act(batchnorm2d(x) + batchnorm2d(xr)) — the ResNet projection block
    output with the shortcut's BN applied inside the same pass (be_bn_attrs
    residual = 2): the shortcut's normalised tensor is never written.  Both
    BNs are train-mode with their own (running) statistics."""
    ins = [x, gamma, beta] + ([running_mean, running_var] if running_mean is not None else [])
    ins += [xr, gamma_r, beta_r, running_mean_r, running_var_r]
    return _op("BATCHNORM2D", ins, L.be_bn_attrs(eps, momentum, int(act), 2))


def bn_conv1x1(x, gamma, beta, running_mean, running_var, w, eps=1e-5, momentum=0.1, act=1):
    """conv1x1(act(batchnorm2d(x)), w) with the normalise + activation applied
    inside the GEMM's operand load (BE_OP_BN_CONV1X1): the BN output never
    reaches HBM.  w: KRSC [K, 1, 1, C]."""
    ins = [x, gamma, beta] + ([running_mean, running_var] if running_mean is not None else []) + [w]
    return _op("BN_CONV1X1", ins, L.be_bn_attrs(eps, momentum, int(act), 0))


def reshape(x, shape):
    a = L.be_shape_attrs(len(shape), (C.c_int64 * 6)(*shape))
    return _op("RESHAPE", [x], a)


def embedding(table, ids):
    return _op("EMBEDDING", [table, ids])


def concat(xs):
    return _op("CONCAT", list(xs))


def sum(x):  # noqa: A001
    return _op("SUM", [x])


def mean(x):
    return _op("MEAN", [x])


def cast(x, dtype):
    return _op("CAST", [x], C.c_int(_dt(dtype)))


def gemm(A, B, D, trans_a=False, trans_b=False, bias=None, act=0, beta=0.0):
    call("be_gemm", A._h, int(trans_a), B._h, int(trans_b), D._h, bias._h if bias is not None else None, int(act),
         C.c_float(beta))


# ------------------------------------------------------------------ autograd / optim
@contextlib.contextmanager
def no_grad():
    v = C.c_int()
    call("be_is_grad_enabled", C.byref(v))
    call("be_set_grad_enabled", 0)
    try:
        yield
    finally:
        call("be_set_grad_enabled", v.value)


def set_compute_dtype(d):
    call("be_set_compute_dtype", _dt(d))


def _handles(ts):
    return (C.c_void_p * len(ts))(*[t._h.value for t in ts])


def sgd_step(params, lr, momentum=0.0, weight_decay=0.0):
    call("be_sgd_step", _handles(params), len(params), C.c_float(lr), C.c_float(momentum), C.c_float(weight_decay))


def sgd_overlap(params, lr=0.0, momentum=0.0, weight_decay=0.0):
    """Register params for the overlapped SGD update inside every later
    backward (be_sgd_overlap); sgd_overlap([]) unregisters."""
    call("be_sgd_overlap", _handles(params) if params else None, len(params), C.c_float(lr), C.c_float(momentum),
         C.c_float(weight_decay))


def sgd_sparse(tables, lr=0.0):
    """Register embedding tables for the touched-rows SGD update applied inside
    the embedding backward (be_sgd_sparse; μ = 0, wd = 0); sgd_sparse([]) unregisters."""
    call("be_sgd_sparse", _handles(tables) if tables else None, len(tables), C.c_float(lr))


def sgd_momentum(param):
    """Copy of the SGD momentum buffer v of `param` (None before the first momentum step)."""
    out = C.c_void_p()
    call("be_sgd_momentum", param._h, C.byref(out))
    return Tensor(out.value) if out.value else None


def zero_grad(params):
    call("be_zero_grad", _handles(params), len(params))


def synchronize():
    call("be_synchronize")


def alloc_stats() -> dict:
    s = L.be_alloc_stats()
    call("be_alloc_stats", C.byref(s))
    return {f: getattr(s, f) for f, _ in L.be_alloc_stats._fields_}


def reset_peak():
    call("be_alloc_reset_peak")


def empty_cache() -> int:
    v = C.c_uint64()
    call("be_empty_cache", C.byref(v))
    return v.value


def round_size(n: int) -> int:
    return int(L.lib().be_round_size(C.c_uint64(n)))


def im2col_offsets(N, C_, H, W, R, S, stride, pad) -> np.ndarray:
    P = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - S) // stride + 1
    out = np.empty((N * P * Q, R * S * C_), np.int64)
    geom = (C.c_int64 * 8)(N, C_, H, W, R, S, stride, pad)
    call("be_debug_im2col_offsets", geom, out.ctypes.data_as(C.POINTER(C.c_int64)))
    return out


def stream_create() -> int:
    v = C.c_uint64()
    call("be_stream_create", C.byref(v))
    return v.value


def event_create() -> int:
    v = C.c_uint64()
    call("be_event_create", C.byref(v))
    return v.value


def event_record(ev: int, stream: int = 0):
    call("be_event_record", C.c_uint64(ev), C.c_uint64(stream))


def stream_wait_event(stream: int, ev: int):
    call("be_stream_wait_event", C.c_uint64(stream), C.c_uint64(ev))


def copy_from_host_on(t: Tensor, src_ptr: int, nbytes: int, stream: int = 0):
    call("be_tensor_copy_from_host_on", t.handle, C.c_void_p(src_ptr), C.c_size_t(nbytes), C.c_uint64(stream))


class InputPipeline:
    """Double-buffered pinned-host → device batch hand-off on a copy stream
    (the data loader's pinned-memory path): batch i+1 is
    copied while step i computes.  `shapes_dtypes` = [(shape, dtype), ...]."""

    def __init__(self, shapes_dtypes):
        self.copy_stream = stream_create()
        self.bufs = [[empty(sh, dt) for sh, dt in shapes_dtypes] for _ in range(2)]
        self.ready = [event_create(), event_create()]
        self.free = [event_create(), event_create()]
        self.primed = [False, False]

    def put(self, slot, host_ptrs_nbytes):
        """Enqueue (non-blocking) the copy of a batch — list of (pinned ptr,
        nbytes) — into buffer `slot`, after its previous user released it."""
        if self.primed[slot]:
            stream_wait_event(self.copy_stream, self.free[slot])
        for t, (ptr, nb) in zip(self.bufs[slot], host_ptrs_nbytes):
            copy_from_host_on(t, ptr, nb, self.copy_stream)
        event_record(self.ready[slot], self.copy_stream)

    def get(self, slot):
        """Tensors of buffer `slot`; the compute stream waits for its copy."""
        stream_wait_event(0, self.ready[slot])
        return self.bufs[slot]

    def release(self, slot):
        """Buffer `slot` is free once the compute work enqueued so far is done."""
        event_record(self.free[slot], 0)
        self.primed[slot] = True


def prof_enable(on=True):
    call("be_prof_enable", int(on))


def prof_read(cap=100000):
    recs = (L.be_prof_rec * cap)()
    n = C.c_int()
    call("be_prof_read", recs, cap, C.byref(n))
    return [dict(name=r.name.decode(), flops=r.flops, bytes=r.bytes, ms=r.ms, m=r.m, n=r.n, k=r.k, t0=r.t_start_ms)
            for r in recs[:n.value]]


# ------------------------------------------------------------------ data parallel
def dist_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    call("be_dist_unique_id", buf)
    return bytes(buf)


def dist_init(rank, world, uid: bytes):
    buf = (C.c_char * 128).from_buffer_copy(uid)
    call("be_dist_init", int(rank), int(world), buf)


def dist_world():
    """(rank, nranks) as the NCCL communicator reports them (ncclCommCount)."""
    r, w = C.c_int(), C.c_int()
    call("be_dist_world", C.byref(r), C.byref(w))
    return r.value, w.value


def p2p_attach(params, rank, world, bucket_bytes=25 << 20) -> bytes:
    """Bucket params for the peer-memory fused allreduce + SGD (be_p2p_attach);
    returns this rank's export blob, to be all-gathered by the caller and
    handed to p2p_connect."""
    cap = 16 + (3 * len(params) + 2) * 64  # header + ≤ 1 + (n + 1) + 2n handles
    buf = (C.c_char * cap)()
    need = C.c_size_t()
    call("be_p2p_attach", _handles(params), len(params), C.c_size_t(bucket_bytes), int(rank), int(world), buf,
         cap, C.byref(need))
    return bytes(buf[:need.value])


def p2p_connect(blobs):
    """blobs: every rank's p2p_attach output, in rank order."""
    n = len(blobs[0])
    assert all(len(b) == n for b in blobs)
    allb = b"".join(blobs)
    call("be_p2p_connect", C.c_char_p(allb), C.c_size_t(n))


def p2p_status() -> int:
    v = C.c_int()
    call("be_p2p_status", C.byref(v))
    return v.value


def ddp_plan(numels, bucket_bytes=25 << 20):
    """Bucket plan of be_ddp_attach (pure host function): (bucket_of, offset_of, bucket_numel)."""
    n = len(numels)
    arr = (C.c_int64 * max(n, 1))(*numels)
    bof = (C.c_int * max(n, 1))()
    off = (C.c_int64 * max(n, 1))()
    bnum = (C.c_int64 * (n + 1))()
    nb = C.c_int()
    call("be_ddp_plan", arr, n, C.c_size_t(bucket_bytes), bof, off, bnum, n + 1, C.byref(nb))
    return list(bof[:n]), list(off[:n]), list(bnum[:nb.value])


def ddp_attach(params, bucket_bytes=25 << 20):
    call("be_ddp_attach", _handles(params), len(params), C.c_size_t(bucket_bytes))


def ddp_detach():
    call("be_ddp_detach")


def ddp_sync_buffers(bufs):
    """Broadcast f32 buffers (BN running statistics) from rank 0."""
    if bufs:
        call("be_ddp_sync_buffers", _handles(bufs), len(bufs))


def dist_world():
    r, w = C.c_int(), C.c_int()
    call("be_dist_world", C.byref(r), C.byref(w))
    return r.value, w.value


def allreduce_(t):
    call("be_allreduce_", t._h)
