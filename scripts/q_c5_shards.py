"""C5 (B=256, T=500, FS ms=5) sharded N ways: the per-rank decode (B/N rows,
utterances [rank*B/N, (rank+1)*B/N)) measured on one B200 for N = 1, 2, 4, 8,
with the full-size fixture parity of the rank's rows.  Ranks share nothing
(no collective), so the N-GPU rate is N x the per-rank rate; the driver's
SCALE run measures the weak-scaling C2 line on real multi-GPU boxes."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_03791_b200 import DecodeAlgo, Model, ModelDims, synth
from paper_2406_03791_b200 import decoders as D
from tests.parity import FullsizeFixture, compare_fullsize
fx = FullsizeFixture("c5")
m = Model.from_seed(ModelDims(1024, 640, 640, 640, 1024, (), "lstm", 2), 1)
T, F = 500, 1024
out = []
for N in (1, 2, 4, 8):
    b0, b1 = 0, 256 // N  # rank 0's shard
    x = synth.uniform(2, (b1 - b0) * T * F, -1.0, 1.0, start=b0 * T * F).reshape(b1 - b0, T, F)
    lens = np.full(b1 - b0, T, np.int32)
    cap = D.build_decode_graph(m, DecodeAlgo.FrameSync, b1 - b0, T, 5, D.Exec.Tensor)
    got = D.replay_decode(cap, x, lens)
    ms = []
    for _ in range(5):
        D.replay_decode(cap, x, lens)
        ms.append(cap.stats()["gpu_ms"])
    sub = FullsizeFixture.__new__(FullsizeFixture); sub.__dict__.update(fx.__dict__)
    sub.counts = fx.counts[b0:b1]; sub.off = fx.off[b0:b1 + 1]
    sub.wins = {(b - b0, i): v for (b, i), v in fx.wins.items() if b0 <= b < b1}
    rep = compare_fullsize(got, sub, f"c5/N{N}")
    per_rank = (b1 - b0) * T / (np.median(ms) / 1000)
    rec = {"n_gpus": N, "rows_per_gpu": b1 - b0, "ms_per_decode": float(np.median(ms)),
           "frames_per_s_per_gpu": per_rank, "projected_frames_per_s": N * per_rank,
           "parity_exact": rep.exact, "parity_near_ties": rep.permitted, "parity_failures": len(rep.failures)}
    print(json.dumps(rec), flush=True)
    out.append(rec)
    cap.close()
json.dump(out, open(os.environ.get("OUT", "gpurun_out/c5_shards.json"), "w"), indent=1)
