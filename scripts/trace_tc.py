"""Event trace of the tensor-core executor on C2 (RNNTG_PROF=1): median
latency between pipeline events over 64 traced joint steps."""
import ctypes as C
import os
import sys

os.environ["RNNTG_PROF"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2406_03791_b200 import DecodeAlgo, Model, synth  # noqa: E402
from paper_2406_03791_b200 import decoders as D  # noqa: E402
from paper_2406_03791_b200._lib import lib  # noqa: E402

dims = D.ModelDims(1024, 640, 640, 640, 1024, (), "lstm", 2)
m = Model.from_seed(dims, 1)
B, T = 32, 250
x = synth.encoder_outputs(2, B, T, 1024)
lens = np.full(B, T, np.int32)
cap = D.build_decode_graph(m, DecodeAlgo.FrameSync, B, T, 5, D.Exec.Tensor)
D.replay_decode(cap, x, lens)
D.replay_decode(cap, x, lens)
st = cap.stats()
print("us/step", 1000 * st["gpu_ms"] / st["joint_evals"])
G = 75
NEV = 136
buf = (C.c_uint64 * ((2 * NEV + G) * 64))()
assert lib().rnntg_debug_trace(cap._h, buf, (2 * NEV + G) * 64) == 0, lib().rnntg_last_error()
allev = np.array(buf, dtype=np.int64).reshape(2 * NEV + G, 64)
cyca = allev[NEV + G:]
ev = allev[:NEV]
names = {0: "J post", 12: "J chunk0 ready", 13: "J chunk9 ready", 1: "J acc ready", 2: "J part pub",
         3: "J decide done", 4: "R0 decide done", 5: "R0 h0 pub", 6: "I1 decide done", 7: "I1 acc ready",
         11: "I1 h1 pub", 10: "R1 decide done", 8: "P decide done", 9: "P acc ready", 14: "P trunk pub",
         16: "J xs written", 17: "J scan done", 18: "J part stored", 22: "R0 part counter", 23: "R0 part staged",
         24: "R0 rules done", 19: "R0 pre ready", 20: "R0 acts in xs", 21: "R0 h stored",
         27: "J mma chunk0 full", 28: "J mma chunk9 full", 29: "J mma issued"}
order = [0, 12, 27, 13, 28, 29, 1, 16, 17, 18, 2, 3, 22, 23, 24, 4, 19, 20, 21, 5, 6, 7, 11, 8, 9, 14]
t0 = ev[0].astype(np.float64)
for e in order:
    d = (ev[e] - ev[0]).astype(np.float64)
    ok = ev[e] > 0
    print(f"{names[e]:18s} +{np.median(d[ok]) / 1000:8.2f} us  (n={ok.sum()})")
step = np.diff(ev[0].astype(np.float64))
print("step period (J post -> next J post):", np.median(step) / 1000, "us")
cyc = np.median((ev[26] - ev[25]).astype(np.float64)); ns = np.median((ev[3] - ev[0]).astype(np.float64))
print("SM clock during decode: %.0f MHz" % (1000 * cyc / ns))
pub = allev[NEV:NEV + G].astype(np.float64) - ev[0][None, :].astype(np.float64)
roles = ["J"] * 9 + ["P"] * 5 + ["R0"] * 20 + ["R1"] * 20 + ["I1"] * 20 + ["E"]
for name in ["J", "R0", "I1", "R1", "P"]:
    idx = [i for i, r in enumerate(roles) if r == name]
    med = [np.median(pub[i]) / 1000 for i in idx]
    print(name, "publish (us after J post, per tile):", " ".join(f"{x:.2f}" for x in med))

print("intra-CTA intervals (clock64, cycles):")
def iv(a, b, name):
    d = (cyca[b] - cyca[a]).astype(np.float64)
    ok = (cyca[a] > 0) & (cyca[b] > 0)
    if ok.any(): print(f"  {name:34s} {np.median(d[ok]):8.0f} cyc")
iv(1, 16, "J acc -> xs written"); iv(16, 17, "J acc -> shuffle argmax done"); iv(17, 18, "J merge -> words stored")
iv(18, 2, "J words -> sumexp published"); iv(2, 3, "J sumexp pub -> decide done")
iv(30, 31, "R0 spin done -> batch done"); iv(31, 22, "R0 batch done -> labels handed"); iv(22, 24, "R0 words seen -> rules done"); iv(24, 4, "R0 rules -> decide done"); iv(4, 19, "R0 decide -> pre ready")
iv(19, 21, "R0 pre -> h stored"); iv(21, 5, "R0 h stored -> h0 published")
iv(23, 24, "R0 (unused)"); iv(6, 7, "I1 decide -> acc ready"); iv(7, 11, "I1 acc -> h1 published"); iv(8, 9, "P decide -> acc ready"); iv(9, 14, "P acc -> trunk published")
iv(9, 32, "P acc -> trunk start"); iv(32, 33, "P trunk compute+stores"); iv(33, 34, "P bump epi_sync"); iv(34, 14, "P release + mark")

print("hand-offs (globaltimer medians relative to J post of the step, us):")
for e, nm in [(40, "P trunk published (prev step)"), (12, "J chunk0 seen"), (41, "R0 decide entered"), (42, "J words stored"), (43, "R0 words seen"), (44, "R0 h0 published"), (48, "I1 chunk0 load issued"), (49, "I1 last chunk load issued"),
                (50, "I1 MMAs issued"), (46, "I1 h1 published"), (51, "P chunk0 load issued"), (52, "P last chunk load issued"),
                (53, "P MMAs issued")]:
    d = (ev[e] - ev[0]).astype(np.float64); ok = ev[e] > 0
    if ok.any(): print(f"  {nm:32s} {np.median(d[ok]) / 1000:8.2f}")
iv(22, 35, "R0 words seen(w0) -> w1 released"); iv(35, 36, "R0 w1 gather issue"); iv(36, 37, "R0 w1 gather -> epi_sync out"); iv(24, 37, "R0 w0 rules done -> epi_sync out (w1)")
np_ = allev[39].astype(np.float64)
print("R0 decide poll iterations per step: median", np.median(np_[np_ > 0]), "min", np_[np_ > 0].min(), "max", np_.max())
l1 = allev[38].astype(np.float64)
print("R0 single strong load latency (cycles): median", np.median(l1[l1 > 0]), "min", l1[l1 > 0].min(), "max", l1.max())
rt = allev[37].astype(np.float64)
if (rt > 0).any() and os.environ.get("RNNTG_ECHO"):
    print("J->R0->J round trip (J clock, cycles): median", np.median(rt[rt > 0]), "min", rt[rt > 0].min())

print("per-chunk pipeline (clock64 cycles after chunk-0 load issue; median):")
for base, nm in [(56, "J"), (92, "I1")]:
    blk = allev[base:base + 35].astype(np.float64)
    ok = blk[0] > 0
    if not ok.any():
        continue
    rel = blk[:, ok] - blk[0, ok][None, :]
    iss = " ".join(f"{np.median(rel[k]):5.0f}" for k in range(10))
    full = " ".join(f"{np.median(rel[10 + k]):5.0f}" for k in range(10))
    print(f"  {nm:3s} load issue: {iss}")
    print(f"  {nm:3s} data full : {full}")
    land = " ".join(f"{np.median(rel[25 + k]):5.0f}" for k in range(10))
    print(f"  {nm:3s} landed    : {land}")
    print(f"  {nm:3s} MMAs issued {np.median(rel[20]):.0f}, acc read {np.median(rel[21]):.0f}, polls after chunk 0 ready: {np.median(blk[22, ok]):.0f}")
    print(f"  {nm:3s} chunk 2: before empty wait {np.median(rel[23]):.0f}, stamp {np.median(rel[2]):.0f}, after TMA issue {np.median(rel[24]):.0f}")
