"""STAMPS build: per-role phase shares of the persistent (tensor) executor's
epilogue thread 0 over one decode (fractions of the kernel's run time)."""
import ctypes as C, os, sys, numpy as np
os.environ["RNNTG_STAMPS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_03791_b200 import DecodeAlgo, Model, ModelDims, synth
from paper_2406_03791_b200 import decoders as D
from paper_2406_03791_b200._lib import lib, check
L = lib()
B = int(os.environ.get("Q_B", "256")); T = int(os.environ.get("Q_T", "100"))
m = Model.from_seed(ModelDims(1024, 640, 640, 640, 1024, (), "lstm", 2), 1)
x = synth.encoder_outputs(2, B, T, 1024); lens = np.full(B, T, np.int32)
cap = D.build_decode_graph(m, DecodeAlgo.FrameSync, B, T, 5, D.Exec.Tensor)
for _ in range(2): D.replay_decode(cap, x, lens)
st = cap.stats()
G = int(os.environ.get("Q_G", "74"))
buf = (C.c_uint64 * (64 * G * 16))()
check(L.rnntg_debug_trace(cap.handle, buf, 64 * G * 16))
a = np.frombuffer(buf, np.uint64).reshape(64, G, 16).astype(np.int64)[63, :, 8:16].astype(np.float64)
print(f"B={B} T={T}: {st['gpu_ms']:.2f} ms, {1000*st['gpu_ms']/st['joint_evals']:.2f} us per group-step")
names = ["load", "J", "decide", "pred", "save", "(wordwait)", "(accwait)"]
roles = [("J", 0, 9), ("P", 9, 14), ("R0", 14, 34), ("R1", 34, 54), ("I1", 54, 74)]
print("role  " + " ".join(f"{n:>10s}" for n in names))
for r, lo, hi in roles:
    tot = a[lo:hi, 7].mean()
    print(f"{r:5s} " + " ".join(f"{a[lo:hi, i].mean() / tot:10.3f}" for i in range(7)))
