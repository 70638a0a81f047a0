"""Profiling driver: one C2 decode, then standalone launches of each decoder
kernel (rnntg_time_kernel).  Run under ncu on the GPU box."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2406_03791_b200 import Model, ModelDims, synth  # noqa: E402
from paper_2406_03791_b200._lib import check, lib  # noqa: E402

cfg = os.environ.get("CFG", "c2")
B, T, ms, algo = {"c2": (32, 250, 5, 0), "c3": (32, 250, 10, 1), "c5": (256, 500, 5, 0)}[cfg]
T = int(os.environ.get("T", T))
dims = ModelDims(1024, 640, 640, 640, 1024, (), "lstm", 2)
m = Model.from_seed(dims, 1)
L = lib()
d = C.c_void_p()
check(L.rnntg_decoder_create(m.handle, algo, int(os.environ.get("EXEC", "0")), B, T, ms, C.byref(d)))
x = synth.encoder_outputs(2, B, T, 1024)
lens = np.full(B, T, np.int32)
check(L.rnntg_bind(d, C.c_void_p(x.ctypes.data), C.c_void_p(lens.ctypes.data)))
for _ in range(int(os.environ.get("DECODES", "1"))):
    check(L.rnntg_launch(d))
check(L.rnntg_sync(d))
reps = int(os.environ.get("REPS", "3"))
for w in [0, 1, 2, 8, 9]:
    ms_ = C.c_float()
    check(L.rnntg_time_kernel(d, w, reps, C.byref(ms_)))
    print(f"kernel {w}: {ms_.value * 1000:.2f} us")
