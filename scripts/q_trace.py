"""CUPTI kernel trace of one decode per executor: kernels, busy, span, per-launch gap."""
import ctypes as C, os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_03791_b200 import DecodeAlgo, Model, ModelDims, synth
from paper_2406_03791_b200 import decoders as D
from paper_2406_03791_b200._lib import lib, check
L = lib()
cfg = os.environ.get("Q_CFG", "c2")
durs = (0, 1, 2, 3, 4) if cfg == "c4" else ()
algo = {"c2": DecodeAlgo.FrameSync, "c3": DecodeAlgo.LabelLoop, "c4": DecodeAlgo.TdtLabelLoop}[cfg]
m = Model.from_seed(ModelDims(1024, 640, 640, 640, 1024, durs, "lstm", 2), 1)
x = synth.encoder_outputs(2, 32, 250, 1024); lens = np.full(32, 250, np.int32)
for ex in [D.Exec[e] for e in sys.argv[1:]] or [D.Exec.Graph]:
    cap = D.build_decode_graph(m, algo, 32, 250, 5 if cfg == "c2" else 10, ex)
    for _ in range(3): D.replay_decode(cap, x, lens)
    st = cap.stats()
    busy, span, nk = C.c_double(), C.c_double(), C.c_int64()
    check(L.rnntg_trace_begin()); cap.launch(); cap.sync(); check(L.rnntg_trace_end(C.byref(busy), C.byref(span), C.byref(nk)))
    print(f"{cfg} {ex.name}: untraced {st['gpu_ms']:.2f} ms ({1000*st['gpu_ms']/st['joint_evals']:.2f} us/step); traced span {span.value:.2f} ms, "
          f"busy {busy.value:.2f} ms, kernels {nk.value}, avg kernel {1000*busy.value/max(nk.value,1):.2f} us, "
          f"gap/launch {1000*(span.value-busy.value)/max(nk.value,1):.2f} us", flush=True)
    cap.close()
