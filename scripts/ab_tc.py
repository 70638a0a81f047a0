"""A/B timing of library variants (RNNTG_LIB) on C2 (AB_CFG=c3/c4 for the
label-looping / TDT configs) with the tensor executor:
median us/step over several decodes, interleaved across variants."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
variants = sys.argv[1:]
code = r'''
import os, sys, numpy as np
sys.path.insert(0, os.environ["ROOT"])
from paper_2406_03791_b200 import DecodeAlgo, Model, synth
from paper_2406_03791_b200 import decoders as D
cfg = os.environ.get("AB_CFG", "c2")
durs = (0, 1, 2, 3, 4) if cfg == "c4" else ()
algo = {"c2": DecodeAlgo.FrameSync, "c3": DecodeAlgo.LabelLoop, "c4": DecodeAlgo.TdtLabelLoop}[cfg]
m = Model.from_seed(D.ModelDims(1024, 640, 640, 640, 1024, durs, "lstm", 2), 1)
x = synth.encoder_outputs(2, 32, 250, 1024); lens = np.full(32, 250, np.int32)
cap = D.build_decode_graph(m, algo, 32, 250, 5 if cfg == "c2" else 10, D.Exec.Tensor)
us = []
for i in range(12):
    D.replay_decode(cap, x, lens); st = cap.stats()
    if i >= 2: us.append(1000 * st["gpu_ms"] / st["joint_evals"])
print("%.3f %.3f" % (np.median(us), np.min(us)))
'''
res = {v: [] for v in variants}
for rep in range(3):
    for v in variants:
        env = dict(os.environ, RNNTG_LIB=f"librnntg_{v}.so", ROOT=ROOT)
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
        res[v].append(line)
for v in variants:
    print(f"{v:12s}", res[v])
