"""Phase profile of the persistent executor (CTA 0, globaltimer), C2 shapes."""
import ctypes as C
import os
import sys

os.environ["RNNTG_PROF"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2406_03791_b200 import Model, ModelDims, synth  # noqa: E402
from paper_2406_03791_b200._lib import Stats, check, lib  # noqa: E402

NAMES = {0: "J pass", 1: "B1 wait", 2: "D decide", 3: "cell0", 4: "B2 wait", 5: "hh0 pass",
         6: "P1 pass", 7: "B3 wait", 8: "Pp pass", 9: "trunk", 10: "B4 wait", 11: "trunk(noacc)",
         12: "B(noacc)"}
os.environ.setdefault("NSLIST", "4,2")
dims = ModelDims(1024, 640, 640, 640, 1024, (), "lstm", 2)
m = Model.from_seed(dims, 1)
L = lib()
B, T = int(os.environ.get("B", 32)), int(os.environ.get("T", 250))
x = synth.encoder_outputs(2, B, T, 1024)
lens = np.full(B, T, np.int32)
for ns in os.environ.get("NSLIST", "2,3").split(","):
    os.environ["RNNTG_NS"] = ns
    d = C.c_void_p()
    check(L.rnntg_decoder_create(m.handle, 0, 1, B, T, 5, C.byref(d)))
    check(L.rnntg_bind(d, C.c_void_p(x.ctypes.data), C.c_void_p(lens.ctypes.data)))
    check(L.rnntg_launch(d))
    check(L.rnntg_sync(d))
    prof = (C.c_uint64 * 16)()
    check(L.rnntg_debug_profile(d, prof))
    check(L.rnntg_launch(d))
    check(L.rnntg_sync(d))
    check(L.rnntg_debug_profile(d, prof))
    st = Stats()
    check(L.rnntg_get_stats(d, C.byref(st)))
    steps = st.joint_evals
    print(f"ns={ns}: {st.gpu_ms:.2f} ms, {steps} steps, {1000 * st.gpu_ms / steps:.2f} us/step")
    tot = sum(prof[i] for i in range(13))
    for i in range(13):
        print(f"   {NAMES[i]:14s} {prof[i] / 1000 / steps:8.2f} us/step  {100 * prof[i] / max(tot, 1):5.1f}%")
    print(f"   copy wait (warp0): {prof[13] / 1000 / steps:.2f} us/step over {prof[14] / steps:.1f} copies; "
          f"reduce+epilogue {prof[15] / 1000 / steps:.2f} us/step")
    check(L.rnntg_decoder_destroy(d))
