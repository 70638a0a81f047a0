"""A/B of library variants (RNNTG_LIB) on one executor: median us/step, interleaved.
    python scripts/ab_exec.py EXEC CFG variant...   (EXEC: Graph, HostLoop, Tensor, ...)"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ex, cfg, variants = sys.argv[1], sys.argv[2], sys.argv[3:]
code = r'''
import os, sys, numpy as np
sys.path.insert(0, os.environ["ROOT"])
from paper_2406_03791_b200 import DecodeAlgo, Model, synth
from paper_2406_03791_b200 import decoders as D
cfg = os.environ["AB_CFG"]
durs = (0, 1, 2, 3, 4) if cfg == "c4" else ()
algo = {"c2": DecodeAlgo.FrameSync, "c3": DecodeAlgo.LabelLoop, "c4": DecodeAlgo.TdtLabelLoop, "c5": DecodeAlgo.FrameSync}[cfg]
B, T = (256, 500) if cfg == "c5" else (32, 250)
m = Model.from_seed(D.ModelDims(1024, 640, 640, 640, 1024, durs, "lstm", 2), 1)
x = synth.encoder_outputs(2, B, T, 1024); lens = np.full(B, T, np.int32)
cap = D.build_decode_graph(m, algo, B, T, 10 if cfg in ("c3", "c4") else 5, D.Exec[os.environ["AB_EXEC"]])
us = []
for i in range(8):
    D.replay_decode(cap, x, lens); st = cap.stats()
    if i >= 2: us.append(1000 * st["gpu_ms"] / st["joint_evals"])
print("%.3f %.3f" % (np.median(us), np.min(us)))
'''
res = {v: [] for v in variants}
for rep in range(3):
    for v in variants:
        env = dict(os.environ, RNNTG_LIB=f"librnntg_{v}.so" if v != "main" else "librnntg.so", ROOT=ROOT, AB_CFG=cfg, AB_EXEC=ex)
        try:
            out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
        except subprocess.TimeoutExpired:
            res[v].append("TIMEOUT"); continue
        res[v].append(out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:])
for v in variants:
    print(f"{ex} {cfg} {v:10s}", res[v], flush=True)
