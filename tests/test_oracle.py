"""The C restatement (oracle/rnnt_oracle.c) against the reference.

Pinned two ways: against the committed golden digests generated from the
unmodified reference decoders (tests/golden/make_golden.py), and -- in the
build container where /root/reference exists -- directly against the
reference library compiled by oracle/Makefile.
"""
import gzip
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json.gz")


@pytest.fixture(scope="module")
def golden():
    with gzip.open(GOLD, "rt") as fh:
        return json.load(fh)


def digest(hyps):
    h = hashlib.sha256()
    for y in hyps:
        h.update(np.int32(len(y.tokens)).tobytes())
        h.update(np.asarray(y.tokens, np.int32).tobytes())
        h.update(np.asarray(y.frames, np.int32).tobytes())
        h.update(np.asarray(y.scores, np.float32).tobytes())
        h.update(np.float64(y.total_score).tobytes())
    return h.hexdigest()


def test_rng_known_answers():
    # splitmix64 (tensor.cpp:633-640) with the published seed-0 first outputs
    r = O.lib()
    import ctypes as C

    class Rng(C.Structure):
        _fields_ = [("state", C.c_uint64)]
    r.orc_rng_next.restype = C.c_uint64
    r.orc_rng_next.argtypes = [C.POINTER(Rng)]
    g = Rng(0)
    assert r.orc_rng_next(C.byref(g)) == 0xE220A8397B1DCDAF
    assert r.orc_rng_next(C.byref(g)) == 0x6E789E6AA1B965F4


def test_random_fs_digests(golden):
    """acceptance.cpp criterion 1 seeds 1..200 (decode_test_util.hpp)."""
    bad = []
    for seed, rec in golden["random"]["fs"].items():
        c = O.random_case(int(seed), False)
        hyps = O.decode_batch(c.dims, c.params, c.x, c.out_len, c.max_symbols, False)
        if digest(hyps) != rec["digest"]:
            bad.append(seed)
    assert not bad


def test_random_tdt_digests(golden):
    """acceptance.cpp criterion 2 seeds 1000..1199."""
    bad = []
    for seed, rec in golden["random"]["tdt"].items():
        c = O.random_case(int(seed), True)
        hyps = O.decode_batch(c.dims, c.params, c.x, c.out_len, c.max_symbols, True)
        if digest(hyps) != rec["digest"]:
            bad.append(seed)
    assert not bad


def test_full_vectors_match(golden):
    for seed, rec in list(golden["random"]["fs"].items())[:12]:
        c = O.random_case(int(seed), False)
        hyps = O.decode_batch(c.dims, c.params, c.x, c.out_len, c.max_symbols, False)
        for h, g in zip(hyps, rec["hyps"]):
            assert h.tokens == g["tokens"] and h.frames == g["frames"]
            assert np.asarray(h.scores, np.float32).view(np.uint32).tolist() == g["scores_hex"]
            assert h.total_score == g["total_score"]


def test_pinned_duration_heads(golden):
    """test_decoders.cpp:351-402: a pinned duration head reduces to LL."""
    for rec in golden["pinned_durations"]:
        d = O.Dims(14, 6, 8, 6, 6, tuple(rec["durations"]))
        p = O.init_params(rec["params_seed"], d)
        p[7][:, :] = -1.0
        p[7][:, 0] = 1.0
        x = O.fill_uniform(rec["x_seed"], -1.0, 1.0, (rec["B"], rec["T"], 6))
        lens = np.array(rec["out_len"], np.int32)
        tdt = O.decode_batch(d, p, x, lens, rec["tdt_ms"], True)
        ll = O.decode_batch(d, p, x, lens, rec["ll_ms"], False)
        assert digest(tdt) == rec["digest"] == digest(ll)


@pytest.mark.parametrize("idx", range(6))
def test_lstm_cases(golden, idx):
    rec = golden["lstm"][idx]
    if rec["name"] == "c1_fs" and os.environ.get("RNNTG_FAST"):
        pytest.skip("slow case")
    d = O.Dims(rec["vocab"], rec["hidden"], rec["hidden"], rec["joint"], rec["feature"],
               tuple(rec["durations"]), O.CELL_LSTM, rec["layers"])
    p = O.init_params(1, d)
    x = O.fill_uniform(2, -1.0, 1.0, (rec["B"], rec["T"], rec["feature"]))
    lens = np.array(rec["out_len"], np.int32)
    hyps = O.decode_batch(d, p, x, lens, rec["ms"], bool(rec["durations"]))
    assert digest(hyps) == rec["digest"]
    st = O.fill_uniform(3, -1.0, 1.0, (2, d.state_width))
    f = O.fill_uniform(4, -1.0, 1.0, (2, rec["feature"]))
    pred = O.prediction(d, p, np.array([0, rec["vocab"]], np.int32), st)
    assert hashlib.sha256(pred.tobytes()).hexdigest() == rec["kat"]["pred_digest"]
    logp, _ = O.joint(d, p, f, pred)
    assert hashlib.sha256(logp.tobytes()).hexdigest() == rec["kat"]["logp_digest"]


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
def test_against_reference_library_directly():
    for seed in (3, 17, 99):
        c = O.random_case(seed, False)
        mine = O.decode_batch(c.dims, c.params, c.x, c.out_len, c.max_symbols, False)
        for algo in ("oracle", "sync_free", "graph_fs", "label_loop", "graph_ll", "baseline"):
            r, _ = O.ref_random_case(seed, False, algo)
            assert O.hyps_equal(mine, r), algo
