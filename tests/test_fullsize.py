"""Full-size parity: every executor against the reference's own scalar oracle
at the BASELINE configs' full sizes (C2 FS ms=5, C3 LL ms=10,
C4 TDT ms=10 at B=32 T=250; C5 FS ms=5 at B=256 T=500; plus the
realistic-emission regime c2b / c3b with a blank-column bias).

The fixtures (tests/golden/fullsize_*.npz) were produced by
tests/golden/make_fullsize.py from the UNMODIFIED reference
(``scalar_reference_decode[_tdt]``, decoders.cpp:670-755) on exactly the
inputs bench.py decodes.  Rule (tests/parity.py): tokens, frames and TDT
durations identical; scores within 1e-4 relative; a divergence is permitted
only where the oracle's top-2 margin in the diverging decision window is
below 1e-4, and every such divergence is counted and printed.
"""
import json
import os

import numpy as np
import pytest

from tests.parity import FullsizeFixture, compare_fullsize

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIGS = ["c2", "c3", "c4", "c5", "c2b", "c3b"]


def _fixture(name):
    path = os.path.join(ROOT, "tests", "golden", f"fullsize_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    return FullsizeFixture(name)


def _inputs(fx):
    from paper_2406_03791_b200 import synth
    B, T, F = fx.meta["B"], fx.meta["T"], fx.meta["dims"]["feature"]
    x = np.empty((B, T, F), np.float32)
    step = 16
    for b0 in range(0, B, step):
        b1 = min(B, b0 + step)
        x[b0:b1] = synth.uniform(2, (b1 - b0) * T * F, -1.0, 1.0, start=b0 * T * F).reshape(b1 - b0, T, F)
    return x, np.full(B, T, np.int32)


# ----------------------------------------------------------------- CPU (no GPU)
@pytest.mark.parametrize("name", CONFIGS)
def test_fixture_consistent(name):
    """The stored vectors hash to the per-utterance digests the generator took
    from the reference's hypotheses (counts, tokens, frames, scores, total)."""
    import hashlib
    fx = _fixture(name)
    assert len(fx.meta["digests"]) == fx.meta["B"] == len(fx.counts)
    for b in range(len(fx.counts)):
        t, f, s, _ = fx.utt(b)
        h = hashlib.sha256()
        h.update(np.int32(len(t)).tobytes())
        h.update(t.astype(np.int32).tobytes())
        h.update(f.astype(np.int32).tobytes())
        h.update(s.astype(np.float32).tobytes())
        h.update(np.float64(fx.totals[b]).tobytes())
        assert h.hexdigest() == fx.meta["digests"][b], (name, b)
        # total_score is the double sum of the scores (decoders.cpp:118-119)
        assert fx.totals[b] == float(np.sum(s.astype(np.float64))) or abs(
            fx.totals[b] - float(np.sum(s.astype(np.float64)))) < 1e-9 * max(1.0, abs(fx.totals[b]))


@pytest.mark.parametrize("name", ["c4", "c2b"])
def test_oracle_reproduces_fixture_utterance(name):
    """The C restatement re-decodes utterance 0 of a full-size config and lands
    on the fixture bit for bit (pins oracle and fixture to each other)."""
    from oracle import oracle as O
    fx = _fixture(name)
    m = fx.meta
    dm = m["dims"]
    d = O.Dims(dm["vocab"], dm["hidden"], dm["hidden"], dm["joint"], dm["feature"], tuple(m["durations"]),
               O.CELL_LSTM, dm["layers"])
    from paper_2406_03791_b200 import synth
    w = synth.init_params(1, synth.param_shapes(dm["vocab"], dm["hidden"], dm["hidden"], dm["joint"],
                                                dm["feature"], tuple(m["durations"]), "lstm", dm["layers"]))
    if m["blank_bias"]:
        w[-2 if m["durations"] else -1][:, dm["vocab"]] += np.float32(m["blank_bias"])
    T, F = m["T"], dm["feature"]
    x = synth.uniform(2, T * F, -1.0, 1.0).reshape(T, F)
    h = O.decode_utt(d, w, x, T, m["ms"], fx.tdt)
    t, f, s, du = fx.utt(0)
    assert list(h.tokens) == t.tolist() and list(h.frames) == f.tolist()
    assert np.asarray(h.scores, np.float32).tobytes() == s.astype(np.float32).tobytes()
    if fx.tdt:
        assert list(h.durations) == du.tolist()


# ------------------------------------------------------------------ GPU parity
EXECS = ["Tensor", "Graph", "Persistent", "HostLoop", "GraphFFMA"]


@pytest.mark.gpu
@pytest.mark.parametrize("exec_name", EXECS)
@pytest.mark.parametrize("name", CONFIGS)
def test_fullsize_parity(name, exec_name):
    from paper_2406_03791_b200 import DecodeAlgo, Model, ModelDims
    from paper_2406_03791_b200 import decoders as D
    fx = _fixture(name)
    m = fx.meta
    dm = m["dims"]
    dims = ModelDims(dm["vocab"], dm["hidden"], dm["hidden"], dm["joint"], dm["feature"],
                     tuple(m["durations"]), "lstm", dm["layers"])
    algo = {"fs": DecodeAlgo.FrameSync, "ll": DecodeAlgo.LabelLoop, "tdt": DecodeAlgo.TdtLabelLoop}[m["algo"]]
    model = Model.from_seed(dims, 1, blank_bias=m["blank_bias"])
    x, lens = _inputs(fx)
    cap = D.build_decode_graph(model, algo, m["B"], m["T"], m["ms"], getattr(D.Exec, exec_name))
    got = D.replay_decode(cap, x, lens)
    stats = cap.stats()
    cap.close()
    model.close()
    rep = compare_fullsize(got, fx, f"{name}/{exec_name}")
    line = {"config": name, "exec": exec_name, "B": m["B"], "T": m["T"], "ms": m["ms"], "algo": m["algo"],
            "utterances": rep.utterances, "exact": rep.exact, "permitted_near_ties": rep.permitted,
            "failures": rep.failures[:5], "max_score_rel": rep.max_score_rel,
            "oracle_decisions": m["decisions"], "oracle_margins_lt_1e-4": m["decisions_margin_lt_1e-4"],
            "tokens": int(sum(len(h.tokens) for h in got)), "stats": stats}
    print("FULLSIZE", json.dumps(line))
    out = os.environ.get("RNNTG_FULLSIZE_LOG")
    if out:
        with open(out, "a") as fh:
            fh.write(json.dumps(line) + "\n")
    assert rep.ok, rep.failures[:5]
