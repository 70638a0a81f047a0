import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_2406_03791_b200 import DecodeAlgo, Model, synth
from paper_2406_03791_b200 import decoders as D
m = Model.from_seed(D.ModelDims(1024, 640, 640, 640, 1024, (), "lstm", 2), 1)
T = int(os.environ.get("T", 20))
x = synth.encoder_outputs(2, 32, T, 1024); lens = np.full(32, T, np.int32)
cap = D.build_decode_graph(m, DecodeAlgo.FrameSync, 32, T, 5, D.Exec.Tensor)
h = D.replay_decode(cap, x, lens)
print("ok", cap.stats(), [len(t.tokens) for t in h[:4]], flush=True)
