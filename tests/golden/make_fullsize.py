"""Full-size parity fixtures: the reference's own scalar oracle on exactly the
inputs bench.py decodes (TEST INFRASTRUCTURE; run in the build container).

    make -f oracle/Makefile && python tests/golden/make_fullsize.py [c2 c3 c4 c5 ...]

For every utterance of a BASELINE config:

* inputs are bench.py's: weights ``init_params(Rng(1))`` (model.cpp:81-108;
  LSTM order per SURVEY App. B) with an optional blank-column bias, encoder
  outputs ``U[-1,1)`` from ``Rng(2)`` over [B,T,F] row-major
  (decode_test_util.hpp:54), out_len = T;
* the UNMODIFIED reference decodes it with ``scalar_reference_decode[_tdt]``
  (decoders.cpp:670-755, via oracle/_ref/librnntsim_ref.so; one utterance per
  worker process);
* the C restatement (oracle/rnnt_oracle.c) decodes it again with every
  decision recorded; its tokens / frames / scores / total must equal the
  reference's bitwise (asserted), so its TDT durations and top-2 margins are
  trusted.

Stored per config (``tests/golden/fullsize_<name>.npz``): counts, tokens,
frames, scores (fp32 bits), totals, TDT durations, and -- sparse -- every
emission window whose minimum oracle top-2 margin (token or duration) is
below 1e-3, which is what the divergence rule of tests/parity.py needs.
"""
from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

OUT = os.path.dirname(os.path.abspath(__file__))
MARGIN_KEEP = 1e-3

# name: (algo, B, T, ms, durations, blank_bias) -- C2 dims (2x640 LSTM, J 640, V 1024, F 1024)
FULL = {
    "c2": ("fs", 32, 250, 5, (), 0.0),
    "c3": ("ll", 32, 250, 10, (), 0.0),
    "c4": ("tdt", 32, 250, 10, (0, 1, 2, 3, 4), 0.0),
    "c5": ("fs", 256, 500, 5, (), 0.0),
    # realistic-emission regime: blank-column bias 0.015 (calibrated on the oracle,
    # C2 dims: ~1.3 tokens/frame at ms=10; raw TDT already emits ~0.8/frame)
    "c2b": ("fs", 32, 250, 5, (), 0.015),
    "c3b": ("ll", 32, 250, 10, (), 0.015),
}
V, H, J, F, L = 1024, 640, 640, 1024, 2

_ctx = {}


def _dims(durs):
    from oracle import oracle as O
    return O.Dims(V, H, H, J, F, tuple(durs), O.CELL_LSTM, L)


def _params(durs, bias):
    from paper_2406_03791_b200 import synth
    w = synth.init_params(1, synth.param_shapes(V, H, H, J, F, durs, "lstm", L))
    if bias:
        w[-2 if durs else -1][:, V] += np.float32(bias)
    return w


def _init(name):
    from oracle import oracle as O
    algo, B, T, ms, durs, bias = FULL[name]
    d = _dims(durs)
    p = _params(durs, bias)
    _ctx.update(name=name, d=d, p=p, m=O.RefModel(d, p))


def _utt(b):
    from oracle import oracle as O
    from paper_2406_03791_b200 import synth
    algo, B, T, ms, durs, bias = FULL[_ctx["name"]]
    tdt = algo == "tdt"
    x = synth.uniform(2, T * F, -1.0, 1.0, start=b * T * F).reshape(T, F)
    t0 = time.time()
    ref, _ = _ctx["m"].decode("oracle_tdt" if tdt else "oracle", x[None], np.array([T], np.int32), ms)
    t1 = time.time()
    orc = O.decode_utt(_ctx["d"], _ctx["p"], x, T, ms, tdt, record=True)
    if not O.hyps_equal(ref, [orc]):
        raise AssertionError(f"{_ctx['name']}[{b}]: C restatement != reference")
    blank = V
    emit = [i for i, dd in enumerate(orc.decisions) if dd[1] != blank]
    # window i = decisions (emit[i-1], emit[i]]; window n = tail after the last emission
    wins = []
    lo = 0
    for i, hi in enumerate(emit + [len(orc.decisions) - 1]):
        w = orc.decisions[lo:hi + 1] or orc.decisions[lo:lo + 1]
        m = min([dd[2] for dd in w] + ([dd[4] for dd in w] if tdt else []), default=np.inf)
        if m < MARGIN_KEEP:
            wins.append((i, m))
        lo = hi + 1
    allm = [dd[2] for dd in orc.decisions]
    return dict(b=b, tokens=np.asarray(orc.tokens, np.int32), frames=np.asarray(orc.frames, np.int32),
                scores=np.asarray(orc.scores, np.float32), total=orc.total_score,
                durs=np.asarray(orc.durations, np.int32), wins=wins, ndec=len(orc.decisions),
                nnear=int(sum(1 for m in allm if m < 1e-4)), minm=float(min(allm)) if allm else np.inf,
                ref_s=t1 - t0)


def digest_utt(tokens, frames, scores, total):
    h = hashlib.sha256()
    h.update(np.int32(len(tokens)).tobytes())
    h.update(np.asarray(tokens, np.int32).tobytes())
    h.update(np.asarray(frames, np.int32).tobytes())
    h.update(np.asarray(scores, np.float32).tobytes())
    h.update(np.float64(total).tobytes())
    return h.hexdigest()


def generate(name, procs):
    algo, B, T, ms, durs, bias = FULL[name]
    t0 = time.time()
    with mp.get_context("fork").Pool(procs, initializer=_init, initargs=(name,)) as pool:
        res = sorted(pool.imap_unordered(_utt, range(B)), key=lambda r: r["b"])
    counts = np.array([len(r["tokens"]) for r in res], np.int32)
    wins = np.array([(r["b"], i, m) for r in res for i, m in r["wins"]],
                    dtype=[("b", np.int32), ("i", np.int32), ("m", np.float32)])
    meta = {"generator": "tests/golden/make_fullsize.py", "config": name, "algo": algo, "B": B,
            "T": T, "ms": ms, "durations": list(durs), "blank_bias": bias,
            "dims": {"vocab": V, "hidden": H, "joint": J, "feature": F, "layers": L, "cell": "lstm"},
            "weights": "init_params(Rng(1)) U[-0.08,0.08)", "x": "Rng(2) U[-1,1) [B,T,F]",
            "out_len": "T", "reference": "scalar_reference_decode%s (decoders.cpp:670-755) via "
            "oracle/_ref; C restatement equal bitwise" % ("_tdt" if algo == "tdt" else ""),
            "decisions": int(sum(r["ndec"] for r in res)),
            "decisions_margin_lt_1e-4": int(sum(r["nnear"] for r in res)),
            "min_margin": float(min(r["minm"] for r in res)),
            "tokens_per_frame": float(counts.sum() / (B * T)),
            "ref_cpu_seconds": float(sum(r["ref_s"] for r in res)),
            "wall_seconds": time.time() - t0,
            "digests": [digest_utt(r["tokens"], r["frames"], r["scores"], r["total"]) for r in res]}
    out = dict(counts=counts, tokens=np.concatenate([r["tokens"] for r in res]).astype(np.int16),
               frames=np.concatenate([r["frames"] for r in res]).astype(np.int16),
               scores=np.concatenate([r["scores"] for r in res]).view(np.uint32),
               totals=np.array([r["total"] for r in res], np.float64), wins=wins,
               meta=np.frombuffer(json.dumps(meta).encode(), np.uint8))
    if algo == "tdt":
        out["durations"] = np.concatenate([r["durs"] for r in res]).astype(np.int8)
    path = os.path.join(OUT, f"fullsize_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: B={B} T={T} ms={ms} tokens/frame {meta['tokens_per_frame']:.2f} "
          f"decisions {meta['decisions']} (<1e-4: {meta['decisions_margin_lt_1e-4']}, min "
          f"{meta['min_margin']:.2g}) windows kept {len(wins)}; {meta['wall_seconds']:.0f}s wall, "
          f"{os.path.getsize(path)} bytes", flush=True)


def main():
    names = sys.argv[1:] or ["c2", "c3", "c4", "c5"]
    procs = int(os.environ.get("PROCS", str(max(1, (os.cpu_count() or 2) - 1))))
    for n in names:
        generate(n, procs)


if __name__ == "__main__":
    main()
