"""One C2 decode with the chosen executor (profiling driver)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2406_03791_b200 import Model, ModelDims, synth  # noqa: E402
from paper_2406_03791_b200._lib import check, lib  # noqa: E402

ex = {"graph": 0, "persistent": 1, "tensor": 2, "hostloop": 3}[sys.argv[1] if len(sys.argv) > 1 else "graph"]
B, T = 32, int(os.environ.get("T", 250))
dims = ModelDims(1024, 640, 640, 640, 1024, (), "lstm", 2)
m = Model.from_seed(dims, 1)
L = lib()
d = C.c_void_p()
check(L.rnntg_decoder_create(m.handle, 0, ex, B, T, 5, C.byref(d)))
x = synth.encoder_outputs(2, B, T, 1024)
lens = np.full(B, T, np.int32)
check(L.rnntg_bind(d, C.c_void_p(x.ctypes.data), C.c_void_p(lens.ctypes.data)))
for _ in range(int(os.environ.get("DECODES", "1"))):
    check(L.rnntg_launch(d))
check(L.rnntg_sync(d))
print("ok")
