"""Quick persistent-executor sanity run (small cases, then one C2 decode)."""
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

for seed, tdt, algo in [(1, False, DecodeAlgo.FrameSync), (2, False, DecodeAlgo.LabelLoop),
                        (1001, True, DecodeAlgo.TdtLabelLoop), (7, False, DecodeAlgo.FrameSync)]:
    c = O.random_case(seed, tdt)
    m = Model(to_model_dims(c.dims), c.params)
    cap = D.build_decode_graph(m, algo, c.x.shape[0], c.x.shape[1], c.max_symbols, D.Exec.Persistent)
    got = D.replay_decode(cap, c.x, c.out_len)
    ref = O.decode_batch(c.dims, c.params, c.x, c.out_len, c.max_symbols, tdt, record=True)
    rep = compare_batch(got, ref, c.dims.vocab, tdt, f"seed{seed}")
    print(seed, algo.name, "ok" if rep.ok else rep.failures, cap.stats(), flush=True)
dims = D.ModelDims(1024, 640, 640, 640, 1024, (), "lstm", 2)
m = Model.from_seed(dims, 1)
B, T = 32, int(os.environ.get("T", 250))
x = synth.encoder_outputs(2, B, T, 1024)
lens = np.full(B, T, np.int32)
for ex in (D.Exec.Persistent, D.Exec.Graph):
    cap = D.build_decode_graph(m, DecodeAlgo.FrameSync, B, T, 5, ex)
    t0 = time.time()
    h = D.replay_decode(cap, x, lens)
    h = D.replay_decode(cap, x, lens)
    st = cap.stats()
    print(ex.name, f"{time.time() - t0:.3f}s", st, "us/step", 1000 * st["gpu_ms"] / st["joint_evals"],
          "frames/s", B * T / (st["gpu_ms"] / 1000), flush=True)
    if ex == D.Exec.Persistent:
        hp = h
    else:
        same = sum(a.tokens == b.tokens and a.frames == b.frames for a, b in zip(h, hp))
        print("graph vs persistent agree:", same, "/", B)
