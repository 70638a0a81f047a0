import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_2406_03791_b200 import DecodeAlgo, Model, ModelDims, synth
from paper_2406_03791_b200 import decoders as D
from tests.parity import FullsizeFixture, compare_fullsize
for name, algo, ms, durs in [("c2", DecodeAlgo.FrameSync, 5, ()), ("c3", DecodeAlgo.LabelLoop, 10, ()), ("c4", DecodeAlgo.TdtLabelLoop, 10, (0,1,2,3,4))]:
    fx = FullsizeFixture(name)
    m = Model.from_seed(ModelDims(1024, 640, 640, 640, 1024, durs, "lstm", 2), 1)
    x = synth.encoder_outputs(2, 32, 250, 1024); lens = np.full(32, 250, np.int32)
    for ex in (D.Exec.Graph, D.Exec.HostLoop, D.Exec.GraphFFMA, D.Exec.Tensor):
        cap = D.build_decode_graph(m, algo, 32, 250, ms, ex)
        got = D.replay_decode(cap, x, lens)
        us = []
        for i in range(4):
            D.replay_decode(cap, x, lens); st = cap.stats(); us.append(1000 * st["gpu_ms"] / st["joint_evals"])
        rep = compare_fullsize(got, fx, name)
        print(name, ex.name, "exact", rep.exact, "perm", rep.permitted, "fail", len(rep.failures), "us/step %.2f" % np.median(us), st, flush=True)
        cap.close()
    m.close()
