"""STAMPS build (RNNTG_STAMPS=1): the per-step chain of the tensor executor at C2,
median over 64 steps of each role's stamp times relative to J's visit start.
Stamps per CTA: 1 J visit start, 3 load done, 4 decision done, 5 pred / idle
done (the role's publish), 6 visit end."""
import ctypes as C, os, sys, numpy as np
os.environ["RNNTG_STAMPS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_03791_b200 import DecodeAlgo, Model, ModelDims, synth
from paper_2406_03791_b200 import decoders as D
from paper_2406_03791_b200._lib import lib, check
L = lib()
m = Model.from_seed(ModelDims(1024, 640, 640, 640, 1024, (), "lstm", 2), 1)
T = 40
x = synth.encoder_outputs(2, 32, T, 1024); lens = np.full(32, T, np.int32)
cap = D.build_decode_graph(m, DecodeAlgo.FrameSync, 32, T, 5, D.Exec.Tensor)
for _ in range(2): D.replay_decode(cap, x, lens)
st = cap.stats()
G = 95
buf = (C.c_uint64 * (64 * G * 16))()
check(L.rnntg_debug_trace(cap.handle, buf, 64 * G * 16))
a = np.frombuffer(buf, np.uint64).reshape(64, G, 16).astype(np.int64)
roles = [("J", 0, 9), ("P", 9, 14), ("R0", 14, 34), ("I0", 34, 54), ("R1", 54, 74), ("I1", 74, 94), ("E", 94, 95)]
t0 = a[:, 0:9, 1].min(axis=1)  # J visit start per step (slot)
ok = t0 > 0
print(f"{1000*st['gpu_ms']/st['joint_evals']:.2f} us/step; per-step times (us) after the J tiles start the step's joint:")
print("role      decide(min/max)      publish(min/max)     end")
for r, lo, hi in roles:
    def med(i, f):
        v = f(a[ok, lo:hi, i], axis=1) - t0[ok]
        return np.median(v) / 1000
    print(f"{r:5s} {med(4, np.min):7.2f} {med(4, np.max):7.2f}   {med(5, np.min):7.2f} {med(5, np.max):7.2f}   {med(6, np.max):7.2f}")
per = np.diff(np.sort(t0[ok])); print("step period median", np.median(per) / 1000)
