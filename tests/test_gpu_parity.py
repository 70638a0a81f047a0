"""GPU parity: the CUDA decoder (through the C ABI) against the CPU oracle.

Mirrors the reference's own decoder tests (tests/test_decoders.cpp,
tests/acceptance.cpp criteria 1-2) with the comparator of tests/parity.py.
"""
import gzip
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.parity import EPS_MARGIN, RTOL, ParityReport, compare_batch, rel_err

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2406_03791_b200")
from paper_2406_03791_b200 import DecodeAlgo, Model, ModelDims  # noqa: E402
from paper_2406_03791_b200 import decoders as D  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json.gz")


def _need_gpu():
    if P._lib.lib().rnntg_device_count() < 1:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200")


def to_model_dims(d: O.Dims) -> ModelDims:
    return ModelDims(d.vocab, d.embed, d.hidden, d.joint, d.feature, tuple(d.durations),
                     "lstm" if d.cell == O.CELL_LSTM else "tanh", d.layers)


@pytest.fixture(scope="module")
def golden():
    with gzip.open(GOLD, "rt") as fh:
        return json.load(fh)


EXECS = [D.Exec.Graph, D.Exec.Persistent, D.Exec.Tensor, D.Exec.HostLoop, D.Exec.GraphFFMA]


def run_case(seed, tdt, algo, report, exec=D.Exec.Graph):
    c = O.random_case(seed, tdt)
    m = Model(to_model_dims(c.dims), c.params)
    ref = O.decode_batch(c.dims, c.params, c.x, c.out_len, c.max_symbols, tdt, record=True)
    cap = D.build_decode_graph(m, algo, c.x.shape[0], c.x.shape[1], c.max_symbols, exec)
    got = D.replay_decode(cap, c.x, c.out_len)
    report.merge(compare_batch(got, ref, c.dims.vocab, tdt, f"seed{seed}/{algo.name}"))
    # replaying the same graph on the same inputs is bit-identical
    again = D.replay_decode(cap, c.x, c.out_len)
    assert all(a == b for a, b in zip(got, again))
    cap.close()
    m.close()
    return got


def test_device_present():
    _need_gpu()


@pytest.mark.parametrize("exec", EXECS, ids=lambda e: e.name)
@pytest.mark.parametrize("algo", [DecodeAlgo.FrameSync, DecodeAlgo.LabelLoop])
def test_random_cases_rnnt(algo, exec):
    """acceptance.cpp criterion 1: seeds 1..200."""
    _need_gpu()
    rep = ParityReport()
    for seed in range(1, 201):
        run_case(seed, False, algo, rep, exec)
    print(f"\n{algo.name}/{exec.name}: {rep.utterances} utts, {rep.exact} exact, {rep.permitted} permitted "
          f"near-tie divergences (eps {EPS_MARGIN}), max score rel {rep.max_score_rel:.2e}")
    assert rep.ok, rep.failures[:5]
    assert rep.permitted <= max(2, rep.utterances // 100)


@pytest.mark.parametrize("exec", EXECS, ids=lambda e: e.name)
def test_random_cases_tdt(exec):
    """acceptance.cpp criterion 2: seeds 1000..1199."""
    _need_gpu()
    rep = ParityReport()
    for seed in range(1000, 1200):
        run_case(seed, True, DecodeAlgo.TdtLabelLoop, rep, exec)
    print(f"\nTDT/{exec.name}: {rep.utterances} utts, {rep.exact} exact, {rep.permitted} permitted")
    assert rep.ok, rep.failures[:5]


def test_pinned_duration_heads(golden):
    """test_decoders.cpp:351-402: TDT with a pinned duration head == label looping."""
    _need_gpu()
    for rec in golden["pinned_durations"]:
        d = O.Dims(14, 6, 8, 6, 6, tuple(rec["durations"]))
        p = O.init_params(rec["params_seed"], d)
        p[7][:, :] = -1.0
        p[7][:, 0] = 1.0
        x = O.fill_uniform(rec["x_seed"], -1.0, 1.0, (rec["B"], rec["T"], 6))
        lens = np.array(rec["out_len"], np.int32)
        m = Model(to_model_dims(d), p)
        tdt = D.tdt_label_looping_decode(m, x, lens, rec["tdt_ms"])
        ll = D.label_looping_decode(m, x, lens, rec["ll_ms"])
        assert [h.tokens for h in tdt] == [h.tokens for h in ll]
        assert [h.frames for h in tdt] == [h.frames for h in ll]
        ref = O.decode_batch(d, p, x, lens, rec["ll_ms"], False, record=True)
        rep = compare_batch(ll, ref, d.vocab, False, "pinned")
        assert rep.ok, rep.failures
        m.close()


@pytest.mark.parametrize("exec", EXECS, ids=lambda e: e.name)
@pytest.mark.parametrize("idx", range(6))
def test_lstm_golden(golden, idx, exec):
    """LSTM configs (C1 dims, C2 dims) against the reference's LstmModel output."""
    _need_gpu()
    rec = golden["lstm"][idx]
    d = O.Dims(rec["vocab"], rec["hidden"], rec["hidden"], rec["joint"], rec["feature"],
               tuple(rec["durations"]), O.CELL_LSTM, rec["layers"])
    p = O.init_params(1, d)
    x = O.fill_uniform(2, -1.0, 1.0, (rec["B"], rec["T"], rec["feature"]))
    lens = np.array(rec["out_len"], np.int32)
    tdt = bool(rec["durations"])
    algo = {"graph_fs": DecodeAlgo.FrameSync, "graph_ll": DecodeAlgo.LabelLoop,
            "graph_tdt": DecodeAlgo.TdtLabelLoop}[rec["algo"]]
    if exec == D.Exec.Persistent and rec["layers"] > 2:
        pytest.skip("persistent executor supports <= 2 layers")
    m = Model(to_model_dims(d), p)
    got = D.replay_decode(D.build_decode_graph(m, algo, rec["B"], rec["T"], rec["ms"], exec), x,
                          lens)
    ref = O.decode_batch(d, p, x, lens, rec["ms"], tdt, record=True)
    # the oracle itself is pinned to the golden reference output
    for h, g in zip(ref, rec["hyps"]):
        assert h.tokens == g["tokens"] and h.frames == g["frames"]
    rep = compare_batch(got, ref, d.vocab, tdt, rec["name"])
    print(f"\n{rec['name']}/{exec.name}: {rep.exact}/{rep.utterances} exact, {rep.permitted} permitted, "
          f"max score rel {rep.max_score_rel:.2e}")
    assert rep.ok, rep.failures


@pytest.mark.parametrize("tdt", [False, True])
def test_tensor_batch_above_kernel_limit(tdt):
    """Tensor executor at B = 80: ONE kernel decoding three balanced row
    groups (27, 27, 26) interleaved; rows keep their order."""
    _need_gpu()
    d = O.Dims(200, 64, 64, 96, 24, (0, 1, 2, 3, 4) if tdt else (), O.CELL_LSTM, 2)
    p = O.init_params(21, d)
    B, T, ms = 80, 12, 3
    x = O.fill_uniform(22, -1.0, 1.0, (B, T, d.feature))
    lens = np.array([T - (5 * i) % 7 for i in range(B)], np.int32)
    algo = DecodeAlgo.TdtLabelLoop if tdt else DecodeAlgo.FrameSync
    m = Model(to_model_dims(d), p)
    cap = D.build_decode_graph(m, algo, B, T, ms, D.Exec.Tensor)
    got = D.replay_decode(cap, x, lens)
    ref = O.decode_batch(d, p, x, lens, ms, tdt, record=True)
    rep = compare_batch(got, ref, d.vocab, tdt, "B80")
    st = cap.stats()
    assert st["emitted"] == sum(len(h.tokens) for h in got)
    print(f"\nB80 tdt={tdt}: {rep.exact}/{rep.utterances} exact, joint evals {st['joint_evals']}")
    assert rep.ok, rep.failures
    m.close()


@pytest.mark.parametrize("H,J,tdt", [(96, 200, False), (320, 640, True), (640, 192, False), (384, 448, True)])
def test_tensor_mixed_chunk_counts(H, J, tdt):
    """Tensor executor with hidden and joint widths padding to different chunk
    counts (the per-CTA weight image is laid out for the larger one; W_lo is
    TMEM-resident for a width-dependent number of leading chunks)."""
    _need_gpu()
    d = O.Dims(300, H, H, J, 40, (0, 1, 2, 3, 4) if tdt else (), O.CELL_LSTM, 2)
    p = O.init_params(11, d)
    B, T, ms = 8, 30, 4
    x = O.fill_uniform(12, -1.0, 1.0, (B, T, d.feature))
    lens = np.array([T - (3 * i) % 9 for i in range(B)], np.int32)
    algo = DecodeAlgo.TdtLabelLoop if tdt else DecodeAlgo.FrameSync
    m = Model(to_model_dims(d), p)
    got = D.replay_decode(D.build_decode_graph(m, algo, B, T, ms, D.Exec.Tensor), x, lens)
    ref = O.decode_batch(d, p, x, lens, ms, tdt, record=True)
    rep = compare_batch(got, ref, d.vocab, tdt, f"mixed H{H} J{J}")
    print(f"\nmixed H{H} J{J}: {rep.exact}/{rep.utterances} exact, max score rel {rep.max_score_rel:.2e}")
    assert rep.ok, rep.failures
    m.close()


@pytest.mark.parametrize("cell,layers,tdt", [("tanh", 1, False), ("lstm", 2, True),
                                              ("lstm", 1, False), ("lstm", 3, True)])
def test_step_joint_and_prediction(cell, layers, tdt):
    """test_model.cpp:224-270 analogue: kernel logits / states vs the oracle."""
    _need_gpu()
    for (V, H, J, F, E) in [(29, 32, 24, 16, 20), (1024, 640, 640, 1024, 640), (7, 5, 4, 3, 6)]:
        if cell == "lstm":
            E = H
        d = O.Dims(V, E, H, J, F, (0, 1, 2, 3, 4) if tdt else (),
                   O.CELL_LSTM if cell == "lstm" else O.CELL_TANH, layers)
        p = O.init_params(3, d)
        m = Model(to_model_dims(d), p)
        B = 37
        st = O.fill_uniform(5, -1.0, 1.0, (B, d.state_width))
        labels = np.array([(i * 7) % (V + 1) for i in range(B)], np.int32)
        got = m.prediction(labels, st)
        ref = O.prediction(d, p, labels, st)
        assert np.max(np.abs(got - ref)) < 2e-5
        f = O.fill_uniform(6, -1.0, 1.0, (B, F))
        off = 0 if cell == "tanh" else 2 * (layers - 1) * H
        g = np.ascontiguousarray(ref[:, off:off + H])
        lg, dl = m.joint(f, g)
        rl, rdl = O.joint(d, p, f, ref)
        assert rel_err(lg, rl) < RTOL, rel_err(lg, rl)
        if tdt:
            assert rel_err(dl, rdl) < RTOL
        m.close()


def test_enc_proj_precision():
    """K1 against a float64 restatement (3xTF32 budget: well inside 1e-4)."""
    _need_gpu()
    d = O.Dims(1024, 640, 640, 640, 1024, (), O.CELL_LSTM, 2)
    p = O.init_params(1, d)
    m = Model(to_model_dims(d), p)
    x = O.fill_uniform(2, -1.0, 1.0, (300, 1024))
    got = m.enc_proj(x)
    ref = x.astype(np.float64) @ p[7].astype(np.float64)
    err = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
    assert err < 1e-5, err
    m.close()


@pytest.mark.parametrize("exec", EXECS, ids=lambda e: e.name)
def test_full_size_properties(exec):
    """C2 (B=32, T=250, 2x640 LSTM, V=1025): properties at full size --
    frame-sync == label-looping bitwise, batch independence, determinism,
    timestamps monotone, counts <= T*ms."""
    _need_gpu()
    dims = ModelDims(1024, 640, 640, 640, 1024, (), "lstm", 2)
    m = Model.from_seed(dims, 1)
    from paper_2406_03791_b200 import synth
    B, T = 32, 250
    x = synth.encoder_outputs(2, B, T, 1024)
    lens = np.full(B, T, np.int32)
    lens[5] = 100
    lens[9] = 0
    fs = D.greedy_decode_sync_free(m, x, lens, 5, exec)
    fs2 = D.greedy_decode_sync_free(m, x, lens, 5, exec)
    assert all(a == b for a, b in zip(fs, fs2))
    ll = D.label_looping_decode(m, x, lens, 5, exec)
    assert all(a.tokens == b.tokens and a.frames == b.frames for a, b in zip(fs, ll))
    for b, h in enumerate(fs):
        assert len(h.tokens) <= lens[b] * 5
        assert all(0 <= t < 1025 - 1 for t in h.tokens)
        assert all(h.frames[i] <= h.frames[i + 1] for i in range(len(h.frames) - 1))
        assert all(0 <= f < max(lens[b], 1) for f in h.frames)
    assert len(fs[9].tokens) == 0
    # batch independence: a sub-batch decodes identically
    sub = D.greedy_decode_sync_free(m, np.ascontiguousarray(x[3:7]), lens[3:7], 5, exec)
    assert all(a == b for a, b in zip(sub, fs[3:7]))
    m.close()


@pytest.mark.parametrize("other", [D.Exec.Persistent, D.Exec.Tensor, D.Exec.HostLoop], ids=lambda e: e.name)
@pytest.mark.parametrize("algo", [DecodeAlgo.FrameSync, DecodeAlgo.LabelLoop], ids=lambda a: a.name)
def test_executors_agree_full_size(other, algo):
    """Graph vs persistent / tensor-core executors on C2 shapes: identical
    token/frame sequences (different summation orders and, for the tensor
    executor, fp16 hi/lo tensor-core products; a near-tie would show here)."""
    _need_gpu()
    dims = ModelDims(1024, 640, 640, 640, 1024, (), "lstm", 2)
    m = Model.from_seed(dims, 1)
    from paper_2406_03791_b200 import synth
    B, T = 32, 250
    x = synth.encoder_outputs(2, B, T, 1024)
    lens = np.full(B, T, np.int32)
    run = D.greedy_decode_sync_free if algo == DecodeAlgo.FrameSync else D.label_looping_decode
    g = run(m, x, lens, 5, D.Exec.Graph)
    p = run(m, x, lens, 5, other)
    same = sum(a.tokens == b.tokens and a.frames == b.frames for a, b in zip(g, p))
    print(f"\nexecutors agree on {same}/{B} utterances")
    assert same == B
    for a, b in zip(g, p):
        assert rel_err(a.scores, b.scores) < RTOL
    m.close()


@pytest.mark.parametrize("B", [33, 96, 256])
@pytest.mark.parametrize("algo", [DecodeAlgo.FrameSync, DecodeAlgo.LabelLoop, DecodeAlgo.TdtLabelLoop],
                         ids=lambda a: a.name)
def test_tensor_row_groups(B, algo):
    """Tensor executor beyond 32 rows in one kernel (ceil(B / 32) row groups,
    every CTA visiting the live groups round-robin): ragged lengths (zeros,
    short rows) so groups finish at different steps; against the oracle."""
    _need_gpu()
    tdt = algo == DecodeAlgo.TdtLabelLoop
    d = O.Dims(150, 64, 64, 96, 24, (0, 1, 2, 3, 4) if tdt else (), O.CELL_LSTM, 2)
    p = O.init_params(31, d)
    T, ms = 14, 3
    x = O.fill_uniform(32, -1.0, 1.0, (B, T, d.feature))
    lens = np.array([0 if i % 29 == 3 else T - (7 * i) % 11 for i in range(B)], np.int32)
    lens[-32:] = np.minimum(lens[-32:], 4)  # the last group finishes early
    m = Model(to_model_dims(d), p)
    cap = D.build_decode_graph(m, algo, B, T, ms, D.Exec.Tensor)
    got = D.replay_decode(cap, x, lens)
    again = D.replay_decode(cap, x, lens)
    assert all(a == b for a, b in zip(got, again))
    ref = O.decode_batch(d, p, x, lens, ms, tdt, record=True)
    rep = compare_batch(got, ref, d.vocab, tdt, f"B{B}/{algo.name}")
    st = cap.stats()
    assert st["emitted"] == sum(len(h.tokens) for h in got)
    print(f"\nB{B}/{algo.name}: {rep.exact}/{rep.utterances} exact, joint evals {st['joint_evals']}")
    assert rep.ok, rep.failures[:5]
    cap.close()
    m.close()


def test_tensor_row_groups_c2_dims():
    """C2 dims (2x640 LSTM, V 1025) at B = 80, T = 6 on the single kernel."""
    _need_gpu()
    d = O.Dims(1024, 640, 640, 640, 1024, (), O.CELL_LSTM, 2)
    p = O.init_params(1, d)
    B, T, ms = 80, 6, 5
    x = O.fill_uniform(2, -1.0, 1.0, (B, T, 1024))
    lens = np.array([T - i % 3 for i in range(B)], np.int32)
    m = Model(to_model_dims(d), p)
    got = D.replay_decode(D.build_decode_graph(m, DecodeAlgo.FrameSync, B, T, ms, D.Exec.Tensor), x, lens)
    ref = O.decode_batch(d, p, x, lens, ms, False, record=True)
    rep = compare_batch(got, ref, d.vocab, False, "c2dims B80")
    print(f"\nc2dims B80: {rep.exact}/{rep.utterances} exact, {rep.permitted} permitted")
    assert rep.ok, rep.failures[:5]
    m.close()


@pytest.mark.parametrize("B,tdt,step", [(8, False, 0), (8, False, 7), (40, False, 7), (8, True, 0)])
def test_tensor_logits_vs_oracle(B, tdt, step):
    """Logit-level parity of the tcgen05 executor (test_model.cpp:224-270
    analogue) at C2 dims: the J tiles' fp32 logits of decision step `step`,
    turned into log-probabilities, against the oracle's joint on the same
    prediction state (replayed from the decoded labels) within 1e-4 relative.
    Random init emits a label at every step (T * ms per row), so at frame-
    looping step s every row is at frame s // ms after s emissions."""
    _need_gpu()
    from paper_2406_03791_b200._lib import check, lib
    durs = (0, 1, 2, 3, 4) if tdt else ()
    d = O.Dims(1024, 640, 640, 640, 1024, durs, O.CELL_LSTM, 2)
    p = O.init_params(1, d)
    T, ms = 4, 5
    x = O.fill_uniform(2, -1.0, 1.0, (B, T, 1024))
    lens = np.full(B, T, np.int32)
    m = Model(to_model_dims(d), p)
    algo = DecodeAlgo.TdtLabelLoop if tdt else DecodeAlgo.FrameSync
    cap = D.build_decode_graph(m, algo, B, T, ms, D.Exec.Tensor)
    hyps = D.replay_decode(cap, x, lens)
    V1, nD = d.vocab + 1, len(durs)
    out = np.zeros((B, V1 + nD), np.float32)
    check(lib().rnntg_debug_logits(cap.handle, step, out.ctypes.data_as(P._lib.C.POINTER(P._lib.C.c_float))))
    # oracle state after `step` emissions (P0 = pred(blank, 0), then the labels)
    st = O.prediction(d, p, np.full(B, d.vocab, np.int32), np.zeros((B, d.state_width), np.float32))
    for k in range(step):
        assert all(len(h.tokens) > k and h.frames[k] == k // ms for h in hyps)
        st = O.prediction(d, p, np.array([h.tokens[k] for h in hyps], np.int32), st)
    f = np.ascontiguousarray(x[:, step // ms, :])
    logp_ref, dlogp_ref = O.joint(d, p, f, st)

    def logsoftmax(v):
        v = v.astype(np.float64)
        mx = v.max(axis=1, keepdims=True)
        return v - (mx + np.log(np.exp(v - mx).sum(axis=1, keepdims=True)))
    logp = logsoftmax(out[:, :V1])
    err = rel_err(logp, logp_ref)
    print(f"\nB{B} tdt={tdt} step {step}: logp rel err {err:.2e}")
    assert err < RTOL, err
    # the emitted label is the argmax of these logits
    if not tdt:
        assert [int(np.argmax(out[b, :V1])) for b in range(B)] == [h.tokens[step] for h in hyps]
    if tdt:
        derr = rel_err(logsoftmax(out[:, V1:]), dlogp_ref)
        print(f"  duration logp rel err {derr:.2e}")
        assert derr < RTOL, derr
    cap.close()
    m.close()


def test_bind_device_lengths_checked_on_device():
    """rnntg_bind_device validates device-resident lengths without a host round
    trip (decoders.cpp:136-140): an out-of-range entry surfaces as
    DimensionError at the next sync, the decoder stays usable afterwards."""
    _need_gpu()
    import torch
    from paper_2406_03791_b200 import errors
    from paper_2406_03791_b200._lib import check, lib
    d = O.Dims(29, 32, 32, 24, 16, (), O.CELL_LSTM, 2)
    p = O.init_params(1, d)
    B, T = 4, 8
    x = O.fill_uniform(2, -1.0, 1.0, (B, T, d.feature))
    m = Model(to_model_dims(d), p)
    cap = D.build_decode_graph(m, DecodeAlgo.FrameSync, B, T, 3, D.Exec.Tensor)
    L = lib()
    xd = torch.from_numpy(x).cuda()
    bad = torch.tensor([8, 9, 3, 0], dtype=torch.int32).cuda()
    check(L.rnntg_bind_device(cap.handle, P._lib.C.c_void_p(xd.data_ptr()), P._lib.C.c_void_p(bad.data_ptr())))
    check(L.rnntg_launch(cap.handle))
    with pytest.raises(errors.DimensionError):
        check(L.rnntg_sync(cap.handle))
    good = np.array([8, 5, 3, 0], np.int32)
    got = D.replay_decode(cap, x, good)
    rep = compare_batch(got, O.decode_batch(d, p, x, good, 3, False, record=True), d.vocab, False, "after")
    assert rep.ok, rep.failures
    cap.close()
    m.close()


@pytest.mark.parametrize("steps", [1, 3])
@pytest.mark.parametrize("algo", [DecodeAlgo.FrameSync, DecodeAlgo.LabelLoop, DecodeAlgo.TdtLabelLoop],
                         ids=lambda a: a.name)
def test_graph_decisions_per_launch(steps, algo):
    """The graph executor's WHILE body with 1 and 3 decisions per kernel-node
    launch (RNNTG_GRAPH_STEPS; the default 16 is covered by the other suites),
    one and two row groups, against the oracle."""
    _need_gpu()
    tdt = algo == DecodeAlgo.TdtLabelLoop
    d = O.Dims(150, 64, 64, 96, 24, (0, 1, 2, 3, 4) if tdt else (), O.CELL_LSTM, 2)
    p = O.init_params(51, d)
    T, ms = 12, 3
    os.environ["RNNTG_GRAPH_STEPS"] = str(steps)
    try:
        for B in (7, 45):
            x = O.fill_uniform(52, -1.0, 1.0, (B, T, d.feature))
            lens = np.array([T - (5 * i) % 7 for i in range(B)], np.int32)
            m = Model(to_model_dims(d), p)
            cap = D.build_decode_graph(m, algo, B, T, ms, D.Exec.Graph)
            got = D.replay_decode(cap, x, lens)
            rep = compare_batch(got, O.decode_batch(d, p, x, lens, ms, tdt, record=True), d.vocab, tdt,
                                f"K{steps}/B{B}")
            assert rep.ok, rep.failures[:5]
            cap.close()
            m.close()
    finally:
        os.environ.pop("RNNTG_GRAPH_STEPS", None)


@pytest.mark.gpu
@pytest.mark.parametrize("algo", [DecodeAlgo.FrameSync, DecodeAlgo.LabelLoop, DecodeAlgo.TdtLabelLoop],
                         ids=lambda a: a.name)
def test_graph_programmatic_dependent_body(algo):
    """RNNTG_GRAPH_PDL=1: the inner WHILE body as two step launches, the
    second a programmatic dependent of the first (prologue before
    griddepcontrol.wait), one and two row groups, against the oracle."""
    _need_gpu()
    tdt = algo == DecodeAlgo.TdtLabelLoop
    d = O.Dims(150, 64, 64, 96, 24, (0, 1, 2, 3, 4) if tdt else (), O.CELL_LSTM, 2)
    p = O.init_params(53, d)
    T, ms = 12, 3
    os.environ["RNNTG_GRAPH_PDL"] = "1"
    os.environ["RNNTG_GRAPH_STEPS"] = "2"
    try:
        for B in (7, 45):
            x = O.fill_uniform(54, -1.0, 1.0, (B, T, d.feature))
            lens = np.array([T - (3 * i) % 7 for i in range(B)], np.int32)
            m = Model(to_model_dims(d), p)
            cap = D.build_decode_graph(m, algo, B, T, ms, D.Exec.Graph)
            got = D.replay_decode(cap, x, lens)
            got2 = D.replay_decode(cap, x, lens)
            rep = compare_batch(got, O.decode_batch(d, p, x, lens, ms, tdt, record=True), d.vocab, tdt, f"PDL/B{B}")
            assert rep.ok, rep.failures[:5]
            assert [h.tokens for h in got2] == [h.tokens for h in got]
            cap.close()
            m.close()
    finally:
        os.environ.pop("RNNTG_GRAPH_PDL", None)
        os.environ.pop("RNNTG_GRAPH_STEPS", None)
