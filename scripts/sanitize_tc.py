"""Small decodes of the tensor-core executor (persistent) and the graph / host
loop on its step kernel, for compute-sanitizer (racecheck / synccheck /
memcheck): python scripts/sanitize_tc.py; checks parity against the oracle."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O
from paper_2406_03791_b200 import DecodeAlgo, Model, ModelDims
from paper_2406_03791_b200 import decoders as D
from tests.parity import compare_batch
# SH: hidden / joint width (512: the smem W_lo image is non-empty, KC 8 > 7 TMEM-resident chunks)
H = int(os.environ.get("SH", "32"))
J = 24 if H == 32 else H
d = O.Dims(29, H, H, J, 16, (0, 1, 2, 3, 4), O.CELL_LSTM, 2)
p = O.init_params(1, d)
B, T = int(os.environ.get("SB", "5")), int(os.environ.get("ST", "8"))
x = O.fill_uniform(2, -1.0, 1.0, (B, T, d.feature))
lens = np.array([T - (3 * i) % 5 for i in range(B)], np.int32)
m = Model(ModelDims(29, H, H, J, 16, (0, 1, 2, 3, 4), "lstm", 2), p, device=0)
execs = [D.Exec[e] for e in os.environ.get("SEXEC", "Tensor,Graph").split(",")]
algos = [(DecodeAlgo.FrameSync, False), (DecodeAlgo.LabelLoop, False), (DecodeAlgo.TdtLabelLoop, True)]
for algo, tdt in algos[:int(os.environ.get("SALGOS", "3"))]:
    for ex in execs:
        cap = D.build_decode_graph(m, algo, B, T, 3, ex)
        got = D.replay_decode(cap, x, lens)
        rep = compare_batch(got, O.decode_batch(d, p, x, lens, 3, tdt, record=True), d.vocab, tdt, algo.name)
        print(algo.name, ex.name, "exact", rep.exact, "/", rep.utterances, "ok", rep.ok, flush=True)
        cap.close()
m.close()
