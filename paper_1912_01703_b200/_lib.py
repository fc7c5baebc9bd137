"""ctypes binding of include/be.h — argument marshalling only.

Every entry point has the same name as in the C header.  Every step of the
training path runs inside libbe.so (sm_100a kernels); this module only
converts Python values into C arguments and raises on non-zero status.  The
library must exist: there is no fallback of any kind.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BE_LIB", os.path.join(_HERE, "libbe.so"))

BE_F32, BE_F64, BE_I64, BE_BOOL, BE_BF16, BE_I32, BE_U8 = 0, 1, 2, 3, 4, 5, 6

ERRORS = {
    1: "BE_E_SHAPE", 2: "BE_E_BROADCAST", 3: "BE_E_DTYPE", 4: "BE_E_AXIS", 5: "BE_E_EMPTY_REDUCTION",
    6: "BE_E_NONCONTIG", 7: "BE_E_VERSION", 8: "BE_E_DOUBLE_BACKWARD", 9: "BE_E_NO_UPSTREAM",
    10: "BE_E_INPLACE_LEAF", 11: "BE_E_MISSING_GRAD", 12: "BE_E_OOM", 13: "BE_E_DOUBLE_FREE",
    14: "BE_E_BAD_HANDLE", 15: "BE_E_CUDA", 16: "BE_E_NCCL", 17: "BE_E_UNSUPPORTED", 18: "BE_E_NOT_INIT",
    19: "BE_E_ARG",
}
OPS = dict(LINEAR=1, MATMUL=2, ADD=3, MUL=4, RELU=5, SOFTMAX_XENT=6, BCE_LOGITS=7, CONV2D=8, MAXPOOL2D=9,
           AVGPOOL_GLOBAL=10, BATCHNORM2D=11, RESHAPE=12, EMBEDDING=13, CONCAT=14, SUM=15, MEAN=16, CAST=17,
           ADD_RELU=18, DROPOUT=19, CONV2D_DEPTHWISE=20, BN_CONV1X1=21)


class BeError(RuntimeError):
    def __init__(self, code, msg):
        self.code = code
        self.name = ERRORS.get(code, str(code))
        super().__init__(f"{self.name}: {msg}")


class be_alloc_stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("raw_alloc_count", "raw_free_count", "cache_hit_count",
                                          "bytes_in_use", "bytes_cached", "peak_bytes_in_use")]


class be_prof_rec(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("flops", C.c_double), ("bytes", C.c_double), ("ms", C.c_float),
                ("m", C.c_int), ("n", C.c_int), ("k", C.c_int), ("t_start_ms", C.c_float)]


class be_linear_attrs(C.Structure):
    _fields_ = [("act", C.c_int), ("out_f32", C.c_int)]


class be_conv_attrs(C.Structure):
    _fields_ = [("stride", C.c_int), ("pad", C.c_int), ("act", C.c_int), ("out_f32", C.c_int), ("bn_stats", C.c_int)]


class be_pool_attrs(C.Structure):
    _fields_ = [("k", C.c_int), ("stride", C.c_int), ("pad", C.c_int)]


class be_bn_attrs(C.Structure):
    _fields_ = [("eps", C.c_float), ("momentum", C.c_float), ("act", C.c_int), ("residual", C.c_int)]


class be_dropout_attrs(C.Structure):
    _fields_ = [("p", C.c_double), ("training", C.c_int), ("seed", C.c_uint64), ("offset", C.c_uint64)]


class be_dwconv_attrs(C.Structure):
    _fields_ = [("stride", C.c_int), ("pad", C.c_int)]


class be_shape_attrs(C.Structure):
    _fields_ = [("rank", C.c_int), ("shape", C.c_int64 * 6)]


RELEASE_CB = C.CFUNCTYPE(None, C.c_void_p)

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_1912_01703_b200.build` "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        T = C.c_void_p
        P = C.POINTER
        sigs = {
            "be_init": [C.c_int, C.c_uint64],
            "be_get_stream": [P(C.c_uint64)],
            "be_launch_count": [P(C.c_uint64)],
            "be_tensor_create": [C.c_void_p, P(C.c_int64), C.c_int, C.c_int, C.c_int, P(T)],
            "be_tensor_empty": [P(C.c_int64), C.c_int, C.c_int, P(T)],
            "be_tensor_from_device": [C.c_void_p, P(C.c_int64), P(C.c_int64), C.c_int, C.c_int, RELEASE_CB,
                                      C.c_void_p, P(T)],
            "be_tensor_to_host": [T, C.c_void_p, C.c_size_t],
            "be_tensor_copy_from_host_async": [T, C.c_void_p, C.c_size_t],
            "be_tensor_copy_to_host_async": [T, C.c_void_p, C.c_size_t],
            "be_tensor_info": [T, P(C.c_int), P(C.c_int64), P(C.c_int64), P(C.c_int), P(C.c_uint64)],
            "be_tensor_version": [T, P(C.c_uint64)],
            "be_tensor_requires_grad": [T, P(C.c_int)],
            "be_retain": [T],
            "be_release": [T],
            "be_fill_": [T, C.c_double],
            "be_copy_": [T, T],
            "be_op": [C.c_int, P(T), C.c_int, C.c_void_p, P(T), C.c_int],
            "be_set_grad_enabled": [C.c_int],
            "be_is_grad_enabled": [P(C.c_int)],
            "be_set_compute_dtype": [C.c_int],
            "be_detach": [T, P(T)],
            "be_backward": [T, T, C.c_int],
            "be_grad": [T, P(T)],
            "be_zero_grad": [P(T), C.c_int],
            "be_sgd_step": [P(T), C.c_int, C.c_float, C.c_float, C.c_float],
            "be_sgd_overlap": [P(T), C.c_int, C.c_float, C.c_float, C.c_float],
            "be_sgd_sparse": [P(T), C.c_int, C.c_float],
            "be_p2p_attach": [P(T), C.c_int, C.c_size_t, C.c_int, C.c_int, C.c_void_p, C.c_size_t, P(C.c_size_t)],
            "be_p2p_connect": [C.c_void_p, C.c_size_t],
            "be_p2p_status": [P(C.c_int)],
            "be_sgd_momentum": [T, P(T)],
            "be_alloc_stats": [P(be_alloc_stats)],
            "be_alloc_reset_peak": [],
            "be_empty_cache": [P(C.c_uint64)],
            "be_record_stream": [T, C.c_uint64],
            "be_raw_alloc": [C.c_uint64, C.c_uint64, P(C.c_uint64)],
            "be_raw_free": [C.c_uint64],
            "be_dist_unique_id": [C.c_void_p],
            "be_dist_init": [C.c_int, C.c_int, C.c_void_p],
            "be_ddp_attach": [P(T), C.c_int, C.c_size_t],
            "be_ddp_detach": [],
            "be_ddp_sync_buffers": [P(T), C.c_int],
            "be_dist_world": [P(C.c_int), P(C.c_int)],
            "be_allreduce_": [T],
            "be_synchronize": [],
            "be_item": [T, P(C.c_double)],
            "be_debug_im2col_offsets": [P(C.c_int64), P(C.c_int64)],
            "be_gemm": [T, C.c_int, T, C.c_int, T, T, C.c_int, C.c_float],
            "be_ddp_plan": [P(C.c_int64), C.c_int, C.c_size_t, P(C.c_int), P(C.c_int64), P(C.c_int64), C.c_int,
                            P(C.c_int)],
            "be_stream_create": [P(C.c_uint64)],
            "be_stream_destroy": [C.c_uint64],
            "be_event_create": [P(C.c_uint64)],
            "be_event_destroy": [C.c_uint64],
            "be_event_record": [C.c_uint64, C.c_uint64],
            "be_stream_wait_event": [C.c_uint64, C.c_uint64],
            "be_tensor_copy_from_host_on": [T, C.c_void_p, C.c_size_t, C.c_uint64],
            "be_prof_enable": [C.c_int],
            "be_prof_read": [P(be_prof_rec), C.c_int, P(C.c_int)],
        }
        for name, args in sigs.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.be_last_error.argtypes = []
        L.be_last_error.restype = C.c_char_p
        L.be_round_size.argtypes = [C.c_uint64]
        L.be_round_size.restype = C.c_uint64
        _lib = L
    return _lib


def check(status):
    if status != 0:
        raise BeError(status, lib().be_last_error().decode(errors="replace"))


def call(name, *args):
    check(getattr(lib(), name)(*args))


EXPORTED = [
    "be_init", "be_get_stream", "be_last_error", "be_launch_count", "be_tensor_create", "be_tensor_empty",
    "be_tensor_from_device", "be_tensor_to_host", "be_tensor_copy_from_host_async", "be_tensor_copy_to_host_async",
    "be_tensor_info", "be_tensor_version", "be_tensor_requires_grad", "be_retain", "be_release", "be_fill_",
    "be_copy_", "be_op", "be_set_grad_enabled", "be_is_grad_enabled", "be_set_compute_dtype", "be_detach",
    "be_backward", "be_grad", "be_zero_grad", "be_sgd_step", "be_alloc_stats", "be_alloc_reset_peak",
    "be_empty_cache", "be_round_size", "be_record_stream", "be_raw_alloc", "be_raw_free", "be_dist_unique_id",
    "be_dist_init", "be_ddp_attach", "be_ddp_detach", "be_allreduce_", "be_synchronize", "be_item",
    "be_debug_im2col_offsets", "be_gemm", "be_prof_enable", "be_prof_read", "be_ddp_plan",
    "be_stream_create", "be_stream_destroy", "be_event_create", "be_event_destroy", "be_event_record",
    "be_stream_wait_event", "be_tensor_copy_from_host_on", "be_sgd_overlap", "be_sgd_sparse", "be_p2p_attach", "be_p2p_connect", "be_p2p_status",
    "be_sgd_momentum", "be_ddp_sync_buffers", "be_dist_world",
]
