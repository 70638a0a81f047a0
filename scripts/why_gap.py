"""Where does bench.py's C2 step time differ from scripts/ab_tc.py's?  One
process, one decoder, timed under different conditions."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2406_03791_b200 import Model, ModelDims, synth  # noqa: E402
from paper_2406_03791_b200 import decoders as D  # noqa: E402
from paper_2406_03791_b200._lib import Stats, check, lib  # noqa: E402

L_ = lib()
dims = ModelDims(1024, 640, 640, 640, 1024, (), "lstm", 2)
mode = sys.argv[1] if len(sys.argv) > 1 else "bench"
if mode == "ab":
    m = Model.from_seed(dims, 1)
else:
    m = Model.from_seed(dims, 1, device=0, blank_bias=0.0)
dh = C.c_void_p()
check(L_.rnntg_decoder_create(m.handle, 0, 2, 32, 250, 5, C.byref(dh)))
x = synth.encoder_outputs(2, 32, 250, 1024)
lens = np.full(32, 250, np.int32)
xd = torch.from_numpy(x).cuda()
ld = torch.from_numpy(lens).cuda()
check(L_.rnntg_bind_device(dh, C.c_void_p(xd.data_ptr()), C.c_void_p(ld.data_ptr())))
stream = torch.cuda.ExternalStream(L_.rnntg_decoder_stream(dh), device=0)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def run(tag, do_flush, n=6):
    out = []
    for i in range(n):
        with torch.cuda.stream(stream):
            if do_flush:
                flush.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
        check(L_.rnntg_launch(dh))
        with torch.cuda.stream(stream):
            b.record(stream)
        check(L_.rnntg_sync(dh))
        torch.cuda.synchronize()
        st = Stats()
        check(L_.rnntg_get_stats(dh, C.byref(st)))
        out.append((a.elapsed_time(b) * 1000 / st.joint_evals, st.gpu_ms * 1000 / st.joint_evals))
    o = np.array(out[1:])
    print(f"{mode:6s} {tag:22s} events {np.median(o[:, 0]):.3f}  own {np.median(o[:, 1]):.3f} us/step")


run("no flush", False)
run("flush", True)
with bench.ClockSampler(0):
    run("flush + smi sampler", True)
run("no flush again", False)
