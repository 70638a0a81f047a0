"""Step-launch stamps (STAMPS=1 build, RNNTG_STAMPS=1): per launch, the kernel
span (first CTA entry .. last CTA end) and the gap to the next launch, plus a
per-role breakdown of one mid-decode launch (C2 role layout)."""
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
for exn in sys.argv[1:] or ["HostLoop", "Graph"]:
    cap = D.build_decode_graph(m, DecodeAlgo.FrameSync, 32, T, 5, D.Exec[exn])
    for _ in range(2): D.replay_decode(cap, x, lens)
    G = int(os.environ.get("Q_G", "74"))
    buf = (C.c_uint64 * (64 * G * 16))()
    check(L.rnntg_debug_trace(cap.handle, buf, 64 * G * 16))
    a = np.frombuffer(buf, np.uint64).reshape(64, G, 16).astype(np.int64)
    st = cap.stats()
    # slots hold steps s = slot (mod 64); the last decode's steps 136..199 fill all slots
    order = sorted(range(64), key=lambda k: a[k, :, 0].min())
    spans, gaps = [], []
    for i, k in enumerate(order):
        spans.append((a[k, :, 7].max() - a[k, :, 0].min()) / 1000)
        if i + 1 < len(order):
            gaps.append((a[order[i + 1], :, 0].min() - a[k, :, 7].max()) / 1000)
    print(f"{exn}: {1000*st['gpu_ms']/st['joint_evals']:.2f} us/step; kernel span median {np.median(spans):.2f} us, "
          f"gap median {np.median(gaps):.2f} us (min {np.min(gaps):.2f})")
    k = order[32]
    t0 = a[k, :, 0].min()
    roles = [("J", 0, 9), ("P", 9, 14), ("R0", 14, 34), ("R1", 34, 54), ("I1", 54, 74)]
    names = ["entry", "-", "run", "load", "decide", "pred", "jtail", "end"]
    print("  role " + " ".join(f"{n:>12s}" for n in names))
    for r, lo, hi in roles:
        row = []
        for i in range(8):
            v = a[k, lo:hi, i]
            v = v[v > 0]
            row.append(f"{(v.min()-t0)/1000:5.1f}-{(v.max()-t0)/1000:5.1f}" if len(v) else "     -      ")
        print(f"  {r:4s} " + " ".join(f"{c:>12s}" for c in row))
    cap.close()
