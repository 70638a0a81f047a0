"""ctypes binding of librnntg.so (include/rnntg.h).

The library is built in-tree by ``make -f paper_2406_03791_b200/csrc/Makefile``
(or ``__graft_entry__.build()``).  There is no fallback: if the shared object
is missing, importing the decoder raises.
"""
import ctypes as C
import os

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
# RNNTG_LIB selects an alternative in-tree build (A/B experiments); default the product library
LIB_PATH = os.path.join(HERE, os.environ.get("RNNTG_LIB", "librnntg.so"))

MAX_DUR = 16


class Dims(C.Structure):
    _fields_ = [("vocab", C.c_int32), ("embed", C.c_int32), ("hidden", C.c_int32),
                ("layers", C.c_int32), ("cell", C.c_int32), ("joint", C.c_int32),
                ("feature", C.c_int32), ("num_durations", C.c_int32),
                ("durations", C.c_int32 * MAX_DUR)]


class Stats(C.Structure):
    _fields_ = [("joint_evals", C.c_int64), ("pred_steps", C.c_int64),
                ("outer_iters", C.c_int64), ("emitted", C.c_int64), ("gpu_ms", C.c_float)]


EXPORTS = [
    "rnntg_last_error", "rnntg_abi_version", "rnntg_device_count", "rnntg_model_create",
    "rnntg_model_destroy", "rnntg_decoder_create", "rnntg_decoder_destroy",
    "rnntg_decoder_capacity", "rnntg_bind", "rnntg_bind_device", "rnntg_launch", "rnntg_sync",
    "rnntg_read", "rnntg_get_stats", "rnntg_decoder_stream", "rnntg_step_joint",
    "rnntg_step_prediction", "rnntg_enc_proj", "rnntg_time_kernel", "rnntg_debug_profile", "rnntg_debug_trace", "rnntg_debug_logits", "rnntg_trace_begin", "rnntg_trace_end",
]

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise errors.CudaError(
            f"{LIB_PATH} is missing: build it with `make -f paper_2406_03791_b200/csrc/Makefile`")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    vp = C.c_void_p
    L.rnntg_last_error.restype = C.c_char_p
    L.rnntg_model_create.argtypes = [C.c_int, P(Dims), P(P(C.c_float)), C.c_int, P(vp)]
    L.rnntg_model_destroy.argtypes = [vp]
    L.rnntg_decoder_create.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P(vp)]
    L.rnntg_decoder_destroy.argtypes = [vp]
    L.rnntg_decoder_capacity.argtypes = [vp]
    L.rnntg_bind.argtypes = [vp, vp, vp]
    L.rnntg_bind_device.argtypes = [vp, vp, vp]
    L.rnntg_launch.argtypes = [vp]
    L.rnntg_sync.argtypes = [vp]
    L.rnntg_read.argtypes = [vp, vp, vp, vp, vp, vp, C.c_int]
    L.rnntg_get_stats.argtypes = [vp, P(Stats)]
    L.rnntg_decoder_stream.restype = vp
    L.rnntg_decoder_stream.argtypes = [vp]
    L.rnntg_step_joint.argtypes = [vp, C.c_int, vp, vp, vp, vp]
    L.rnntg_step_prediction.argtypes = [vp, C.c_int, vp, vp, vp]
    L.rnntg_enc_proj.argtypes = [vp, C.c_int, vp, vp]
    L.rnntg_time_kernel.argtypes = [vp, C.c_int, C.c_int, P(C.c_float)]
    L.rnntg_debug_profile.argtypes = [vp, P(C.c_uint64)]
    L.rnntg_debug_trace.argtypes = [vp, P(C.c_uint64), C.c_int]
    L.rnntg_debug_logits.argtypes = [vp, C.c_int, P(C.c_float)]
    L.rnntg_trace_end.argtypes = [P(C.c_double), P(C.c_double), P(C.c_int64)]
    _lib = L
    return L


def check(status: int):
    if status != 0:
        msg = lib().rnntg_last_error().decode(errors="replace")
        raise errors.STATUS.get(status, errors.Error)(msg)
