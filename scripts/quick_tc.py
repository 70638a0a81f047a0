"""Tensor-core persistent executor sanity run: small oracle cases, then C2."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2406_03791_b200 import DecodeAlgo, Model, synth  # noqa: E402
from paper_2406_03791_b200 import decoders as D  # noqa: E402
from tests.parity import compare_batch  # noqa: E402
from tests.test_gpu_parity import to_model_dims  # noqa: E402

EX = D.Exec.Tensor
nseeds = int(os.environ.get("NSEEDS", 4))
for seed0, tdt, algo in [(1, False, DecodeAlgo.FrameSync), (2, False, DecodeAlgo.LabelLoop),
                         (1001, True, DecodeAlgo.TdtLabelLoop)]:
    for seed in range(seed0, seed0 + nseeds):
        c = O.random_case(seed, tdt)
        m = Model(to_model_dims(c.dims), c.params)
        try:
            cap = D.build_decode_graph(m, algo, c.x.shape[0], c.x.shape[1], c.max_symbols, EX)
        except Exception as e:  # noqa: BLE001
            print(seed, algo.name, "skip:", e, flush=True)
            continue
        got = D.replay_decode(cap, c.x, c.out_len)
        ref = O.decode_batch(c.dims, c.params, c.x, c.out_len, c.max_symbols, tdt, record=True)
        rep = compare_batch(got, ref, c.dims.vocab, tdt, f"seed{seed}")
        print(seed, algo.name, c.dims, c.x.shape, "ok" if rep.ok else rep.failures[:3],
              f"exact {rep.exact}/{rep.utterances} maxerr {rep.max_score_rel:.2e}", cap.stats(), flush=True)
dims = D.ModelDims(1024, 640, 640, 640, 1024, (), "lstm", 2)
m = Model.from_seed(dims, 1)
B, T = 32, int(os.environ.get("T", 250))
x = synth.encoder_outputs(2, B, T, 1024)
lens = np.full(B, T, np.int32)
res = {}
for ex in (EX, D.Exec.Persistent):
    cap = D.build_decode_graph(m, DecodeAlgo.FrameSync, B, T, 5, ex)
    t0 = time.time()
    h = D.replay_decode(cap, x, lens)
    h = D.replay_decode(cap, x, lens)
    st = cap.stats()
    print(ex.name, f"{time.time() - t0:.3f}s", st, "us/step", 1000 * st["gpu_ms"] / st["joint_evals"],
          "frames/s", B * T / (st["gpu_ms"] / 1000), flush=True)
    res[ex] = h
a, b = res[EX], res[D.Exec.Persistent]
same = sum(p.tokens == q.tokens and p.frames == q.frames for p, q in zip(a, b))
maxd = max((float(np.max(np.abs(np.asarray(p.scores) - np.asarray(q.scores)))) if (p.tokens == q.tokens and len(p.scores)) else 0.0)
           for p, q in zip(a, b))
print("tensor vs persistent agree:", same, "/", B, "max score diff", maxd)
