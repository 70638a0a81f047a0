"""Generate the golden parity fixtures from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/librnntsim_ref.so, i.e. the
reference compiled from /root/reference/proj/src by oracle/Makefile):

    make -f oracle/Makefile && python tests/golden/make_golden.py

Everything written here comes out of the reference's own decoders
(decoders.cpp) and models (NeuralModel, plus the LstmModel oracle extension
in oracle/ref_capi.cpp), so the committed files pin the C restatement and
the CUDA decoder to the reference without needing /root/reference at test
time.  Inputs are regenerated from splitmix64 seeds (tensor.cpp:633-653;
decode_test_util.hpp:38-59), so only outputs are stored.
"""
import gzip
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def digest(hyps):
    h = hashlib.sha256()
    for y in hyps:
        h.update(np.int32(len(y.tokens)).tobytes())
        h.update(np.asarray(y.tokens, np.int32).tobytes())
        h.update(np.asarray(y.frames, np.int32).tobytes())
        h.update(np.asarray(y.scores, np.float32).tobytes())
        h.update(np.float64(y.total_score).tobytes())
    return h.hexdigest()


def hyp_json(hyps):
    return [{"tokens": list(map(int, y.tokens)), "frames": list(map(int, y.frames)),
             "scores_hex": np.asarray(y.scores, np.float32).view(np.uint32).tolist(),
             "total_score": float(y.total_score)} for y in hyps]


def random_cases():
    out = {"fs": {}, "tdt": {}}
    for seed in range(1, 201):
        ref, je = O.ref_random_case(seed, False, "graph_fs")
        for algo in ("oracle", "baseline", "sync_free", "label_loop", "graph_ll"):
            other, _ = O.ref_random_case(seed, False, algo)
            assert O.hyps_equal(ref, other), (seed, algo)
        rec = {"digest": digest(ref), "fs_joint_evals": je}
        if seed <= 12:
            rec["hyps"] = hyp_json(ref)
        out["fs"][str(seed)] = rec
    for seed in range(1000, 1200):
        ref, je = O.ref_random_case(seed, True, "graph_tdt")
        for algo in ("oracle_tdt", "tdt"):
            other, _ = O.ref_random_case(seed, True, algo)
            assert O.hyps_equal(ref, other), (seed, algo)
        rec = {"digest": digest(ref)}
        if seed < 1012:
            rec["hyps"] = hyp_json(ref)
        out["tdt"][str(seed)] = rec
    return out


def pinned_duration_cases():
    """acceptance.cpp:147-186 / test_decoders.cpp:351-402: a duration head
    pinned to class 0 decodes like label looping."""
    res = []
    for (durs, pseed, xseed, B, T, lens, ms_list, ll_ms) in [
            ((0, 1, 2, 3, 4), 31337, 31338, 4, 12, [12, 9, 12, 4], [1, 2, 5], None),
            ((1, 2, 3, 4), 41414, 41415, 3, 10, [10, 7, 10], [4], 1)]:
        d = O.Dims(14, 6, 8, 6, 6, durs)
        p = O.init_params(pseed, d)
        dur = p[7]
        dur[:, :] = -1.0
        dur[:, 0] = 1.0
        x = O.fill_uniform(xseed, -1.0, 1.0, (B, T, d.feature))
        lens = np.array(lens, np.int32)
        m = O.RefModel(d, p)
        for ms in ms_list:
            tdt, _ = m.decode("tdt", x, lens, ms)
            ll, _ = m.decode("label_loop", x, lens, ll_ms or ms)
            assert O.hyps_equal(tdt, ll)
            res.append({"durations": list(durs), "params_seed": pseed, "x_seed": xseed,
                        "B": B, "T": T, "out_len": lens.tolist(), "tdt_ms": ms,
                        "ll_ms": ll_ms or ms, "digest": digest(tdt), "hyps": hyp_json(tdt)})
    return res


LSTM_CASES = [
    # name, vocab, hidden, joint, feature, layers, durations, B, T, ms, algo
    ("c1_fs", 128, 320, 320, 256, 1, (), 4, 200, 5, "graph_fs"),
    ("c2dims_fs", 1024, 640, 640, 1024, 2, (), 2, 6, 5, "graph_fs"),
    ("c2dims_ll", 1024, 640, 640, 1024, 2, (), 2, 6, 10, "graph_ll"),
    ("c2dims_tdt", 1024, 640, 640, 1024, 2, (0, 1, 2, 3, 4), 2, 10, 10, "graph_tdt"),
    ("small_lstm_tdt", 29, 32, 24, 16, 2, (0, 1, 2, 3, 4), 5, 16, 3, "graph_tdt"),
    ("small_lstm_fs", 29, 32, 24, 16, 3, (), 5, 16, 3, "graph_fs"),
]


def lstm_cases():
    res = []
    for name, V, H, J, F, L, durs, B, T, ms, algo in LSTM_CASES:
        d = O.Dims(V, H, H, J, F, durs, O.CELL_LSTM, L)
        p = O.init_params(1, d)
        x = O.fill_uniform(2, -1.0, 1.0, (B, T, F))
        lens = np.full(B, T, np.int32)
        if B > 2:
            lens[1] = T // 2
            lens[-1] = 0 if B > 3 else T
        m = O.RefModel(d, p)
        hyps, secs = m.decode(algo, x, lens, ms, threads=min(B, 8))
        # joint / prediction KAT on the same model
        st = O.fill_uniform(3, -1.0, 1.0, (2, d.state_width))
        f = O.fill_uniform(4, -1.0, 1.0, (2, F))
        lab = np.array([0, V], np.int32)
        pred = m.prediction(lab, st)
        logp, dlogp = m.joint(f, pred)
        res.append({"name": name, "vocab": V, "hidden": H, "joint": J, "feature": F,
                    "layers": L, "durations": list(durs), "B": B, "T": T, "ms": ms,
                    "algo": algo, "out_len": lens.tolist(), "digest": digest(hyps),
                    "hyps": hyp_json(hyps),
                    "kat": {"pred_digest": hashlib.sha256(pred.tobytes()).hexdigest(),
                            "logp_hex": logp.view(np.uint32).tolist() if V < 200 else None,
                            "logp_digest": hashlib.sha256(logp.tobytes()).hexdigest(),
                            "dur_logp_hex": dlogp.view(np.uint32).tolist() if dlogp is not None else None},
                    "ref_seconds": secs})
        print(name, [len(h.tokens) for h in hyps], f"{secs:.1f}s", flush=True)
    return res


def main():
    data = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/proj",
            "random": random_cases(), "pinned_durations": pinned_duration_cases(),
            "lstm": lstm_cases()}
    path = os.path.join(OUT, "reference_golden.json.gz")
    with gzip.open(path, "wt") as fh:
        json.dump(data, fh, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
