"""RNNTG_PROF=1 event trace of the tensor executor at C2 (single group): the
per-step hand-off chain in globaltimer ns (cross-CTA) and the J / I_1 tracer
CTAs' per-chunk load / MMA times in clock64 cycles (same SM), medians over the
traced window (steps 100..163)."""
import ctypes as C, os, sys, numpy as np
os.environ["RNNTG_PROF"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_03791_b200 import DecodeAlgo, Model, ModelDims, synth
from paper_2406_03791_b200 import decoders as D
from paper_2406_03791_b200._lib import lib, check
L = lib()
NEV, WIN = 136, 64
m = Model.from_seed(ModelDims(1024, 640, 640, 640, 1024, (), "lstm", 2), 1)
T = 40
x = synth.encoder_outputs(2, 32, T, 1024); lens = np.full(32, T, np.int32)
cap = D.build_decode_graph(m, DecodeAlgo.FrameSync, 32, T, 5, D.Exec.Tensor)
for _ in range(2): D.replay_decode(cap, x, lens)
st = cap.stats()
G = 95
n = (2 * NEV + G) * WIN
buf = (C.c_uint64 * n)()
check(L.rnntg_debug_trace(cap.handle, buf, n))
a = np.frombuffer(buf, np.uint64).reshape(2 * NEV + G, WIN).astype(np.int64)
gt = a[:NEV]; pub = a[NEV:NEV + G]; ck = a[NEV + G:]
print(f"{1000*st['gpu_ms']/st['joint_evals']:.2f} us/step (traced build)")
s = np.arange(1, WIN - 1)
ref = gt[42, s]  # J tracer: step s words stored
def rel(v):
    v = v - ref
    return np.median(v) / 1000.0
print("globaltimer, us relative to J's words of step s (J tracer, first J CTA):")
rows = [("J words s (42)", gt[42, s]), ("I1 chunk0 issue (48)", gt[48, s]), ("I1 last chunk issue (49)", gt[49, s]),
        ("I1 MMA issued (50)", gt[50, s]), ("I1 h1 published (46)", gt[46, s]),
        ("P chunk0 issue (51)", gt[51, s]), ("P last chunk issue (52)", gt[52, s]), ("P MMA issued (53)", gt[53, s]),
        ("P trunk published (40)", gt[40, s]), ("J words s+1 (42)", gt[42, s + 1])]
for name, v in rows:
    print(f"  {name:28s} {rel(v):7.2f}")
print("all CTAs' publish (mark_pub) of step s, min / median / max per role:")
roles = [("J", 0, 9), ("P", 9, 14), ("R0", 14, 34), ("I0", 34, 54), ("R1", 54, 74), ("I1", 74, 94)]
for r, lo, hi in roles:
    v = pub[lo:hi][:, s] - ref[None, :]
    print(f"  {r:3s} {np.median(v.min(0))/1000:7.2f} {np.median(np.median(v, 0))/1000:7.2f} {np.median(v.max(0))/1000:7.2f}")
def chunks(ev0, base_ev, name):
    base = ck[base_ev, s]
    iss = [np.median(gt[ev0 + k, s] - base) for k in range(10)]  # (log_chunks: clock64 in the event rows)
    full = [np.median(gt[ev0 + 10 + k, s] - base) for k in range(10)]
    land = [np.median(gt[ev0 + 25 + k, s] - base) for k in range(10)]
    print(f"{name} (clock64 cycles rel. to its mark {base_ev}):")
    print("  issue  " + " ".join(f"{x:6.0f}" for x in iss))
    print("  landed " + " ".join(f"{x:6.0f}" for x in land))
    print("  full   " + " ".join(f"{x:6.0f}" for x in full))
    print(f"  MMA issued {np.median(gt[ev0 + 20, s] - base):.0f}  acc read {np.median(gt[ev0 + 21, s] - base):.0f}  "
          f"polls after chunk0 {np.median(gt[ev0 + 22, s]):.0f}")
chunks(56, 0, "J tracer")
print("  J marks: acc ready(1) %.0f  argmax(17) %.0f  word(18) %.0f  end(2) %.0f" % tuple(
    np.median(ck[e, s] - ck[0, s]) for e in (1, 17, 18, 2)))
chunks(92, 7, "I1 tracer")
print("  I1: acc read(7) -> h1 published(11) %.0f cycles" % np.median(ck[11, s] - ck[7, s]))
print("  P: acc read(9) -> trunk start(32) %.0f, -> staged(33) %.0f, -> published(14) %.0f cycles" % tuple(
    np.median(ck[e, s] - ck[9, s]) for e in (32, 33, 14)))
cap.close()
