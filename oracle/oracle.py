"""ctypes view of the parity checkers (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU arms may import this
module.  It loads

* ``oracle/liboracle.so`` -- the plain-C restatement of the reference path
  (oracle/rnnt_oracle.c), and
* ``oracle/_ref/librnntsim_ref.so`` -- the unmodified reference decoders
  compiled from /root/reference/proj/src (oracle/Makefile), when present.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "librnntsim_ref.so")

CELL_TANH, CELL_LSTM = 0, 1
MAX_DUR = 16


class OrcDims(C.Structure):
    _fields_ = [("vocab", C.c_int32), ("embed", C.c_int32), ("hidden", C.c_int32),
                ("layers", C.c_int32), ("cell", C.c_int32), ("joint", C.c_int32),
                ("feature", C.c_int32), ("num_durations", C.c_int32),
                ("durations", C.c_int32 * MAX_DUR)]


class OrcDecision(C.Structure):
    _fields_ = [("t", C.c_int32), ("k", C.c_int32), ("dur_idx", C.c_int32),
                ("dur", C.c_int32), ("v", C.c_float), ("margin", C.c_float),
                ("dur_margin", C.c_float)]


@dataclass
class Dims:
    """RnntDims (model.hpp:31-40) plus the LSTM extension (cell, layers)."""
    vocab: int
    embed: int
    hidden: int
    joint: int
    feature: int
    durations: tuple = ()
    cell: int = CELL_TANH
    layers: int = 1

    def to_c(self) -> OrcDims:
        d = OrcDims(self.vocab, self.embed, self.hidden, self.layers, self.cell,
                    self.joint, self.feature, len(self.durations))
        for i, v in enumerate(self.durations):
            d.durations[i] = v
        return d

    @property
    def state_width(self) -> int:
        return self.hidden if self.cell == CELL_TANH else 2 * self.layers * self.hidden


@dataclass
class Hyp:
    tokens: list
    frames: list
    scores: list           # float32 values
    total_score: float
    durations: list = field(default_factory=list)
    decisions: list = field(default_factory=list)  # (t, k, margin, dur, dur_margin)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -f oracle/Makefile`")
        L = C.CDLL(ORACLE_SO)
        P = C.POINTER
        L.orc_num_params.argtypes = [P(OrcDims)]
        L.orc_param_size.argtypes = [P(OrcDims), C.c_int, P(C.c_int64), P(C.c_int64)]
        L.orc_init_params.argtypes = [C.c_uint64, P(OrcDims), P(P(C.c_float))]
        L.orc_validate_dims.argtypes = [P(OrcDims)]
        L.orc_prediction.argtypes = [P(OrcDims), P(P(C.c_float)), C.c_int, P(C.c_int32),
                                     P(C.c_float), P(C.c_float)]
        L.orc_joint.argtypes = [P(OrcDims), P(P(C.c_float)), C.c_int, P(C.c_float),
                                P(C.c_float), C.c_int64, P(C.c_float), P(C.c_float)]
        L.orc_decode_utt.argtypes = [P(OrcDims), P(P(C.c_float)), P(C.c_float), C.c_int,
                                     C.c_int, C.c_int, C.c_int, P(C.c_int32), P(C.c_int32),
                                     P(C.c_float), P(C.c_int32), C.c_int, P(OrcDecision),
                                     C.c_int, P(C.c_int), P(C.c_double)]
        L.orc_random_case_header.restype = C.c_uint64
        L.orc_random_case_header.argtypes = [C.c_uint64, C.c_int, P(OrcDims), P(C.c_int),
                                             P(C.c_int), P(C.c_int)]
        L.orc_random_case_inputs.argtypes = [C.c_uint64, P(C.c_float), P(C.c_int32)]
        L.orc_fill_uniform.argtypes = [C.c_uint64, C.c_float, C.c_float, P(C.c_float),
                                       C.c_int64]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"{REF_SO} missing (reference not built)")
        R = C.CDLL(REF_SO)
        P = C.POINTER
        R.ref_last_error.restype = C.c_char_p
        R.ref_random_case_decode.argtypes = [C.c_uint64, C.c_int, C.c_int, P(C.c_int32),
                                             P(C.c_int32), P(C.c_int32), P(C.c_float),
                                             P(C.c_double), C.c_int, P(C.c_int64)]
        R.ref_random_case_params.argtypes = [C.c_uint64, C.c_int, P(P(C.c_float))]
        R.ref_model_create.restype = C.c_void_p
        R.ref_model_create.argtypes = [P(OrcDims), P(P(C.c_float))]
        R.ref_model_destroy.argtypes = [C.c_void_p]
        R.ref_decode.argtypes = [C.c_void_p, C.c_int, P(C.c_float), C.c_int, C.c_int,
                                 P(C.c_int32), C.c_int, C.c_int, P(C.c_int32), P(C.c_int32),
                                 P(C.c_int32), P(C.c_float), P(C.c_double), C.c_int,
                                 P(C.c_double)]
        R.ref_joint.argtypes = [C.c_void_p, C.c_int, P(C.c_float), P(C.c_float),
                                P(C.c_float), P(C.c_float)]
        R.ref_prediction.argtypes = [C.c_void_p, C.c_int, P(C.c_int32), P(C.c_float),
                                     P(C.c_float)]
        _ref = R
    return _ref


def _fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _ptr_array(arrs):
    arr = (C.POINTER(C.c_float) * len(arrs))()
    for i, a in enumerate(arrs):
        arr[i] = _fp(a)
    return arr


def param_shapes(d: Dims):
    cd = d.to_c()
    n = lib().orc_num_params(C.byref(cd))
    out = []
    for i in range(n):
        r, c = C.c_int64(), C.c_int64()
        lib().orc_param_size(C.byref(cd), i, C.byref(r), C.byref(c))
        out.append((r.value, c.value))
    return out


def init_params(seed: int, d: Dims):
    """init_params (model.cpp:81-108; LSTM extension keeps the same order)."""
    shapes = param_shapes(d)
    arrs = [np.zeros(s, dtype=np.float32) for s in shapes]
    cd = d.to_c()
    if lib().orc_init_params(seed, C.byref(cd), _ptr_array(arrs)) != 0:
        raise ValueError("invalid dims")
    return arrs


def fill_uniform(seed: int, lo: float, hi: float, shape):
    n = int(np.prod(shape))
    a = np.zeros(n, dtype=np.float32)
    lib().orc_fill_uniform(seed, lo, hi, _fp(a), n)
    return a.reshape(shape)


@dataclass
class RandomCase:
    seed: int
    dims: Dims
    params: list
    x: np.ndarray
    out_len: np.ndarray
    max_symbols: int


def random_case(seed: int, with_durations: bool) -> RandomCase:
    """make_random_case (decode_test_util.hpp:38-59)."""
    cd = OrcDims()
    b, t, ms = C.c_int(), C.c_int(), C.c_int()
    pseed = lib().orc_random_case_header(seed, int(with_durations), C.byref(cd),
                                         C.byref(b), C.byref(t), C.byref(ms))
    d = Dims(cd.vocab, cd.embed, cd.hidden, cd.joint, cd.feature,
             tuple(cd.durations[i] for i in range(cd.num_durations)), cd.cell, cd.layers)
    x = np.zeros((b.value, t.value, d.feature), dtype=np.float32)
    lens = np.zeros(b.value, dtype=np.int32)
    lib().orc_random_case_inputs(seed, _fp(x), _ip(lens))
    return RandomCase(seed, d, init_params(pseed, d), x, lens, ms.value)


def decode_utt(d: Dims, params, feats, out_len, ms, tdt, record=False) -> Hyp:
    """scalar_reference_decode[_tdt] (decoders.cpp:670-755) on one utterance."""
    feats = np.ascontiguousarray(feats, dtype=np.float32)
    T = feats.shape[0]
    if tdt:
        # TDT may emit up to ms per frame index and skip; bound generously
        cap = max(1, T * ms + 1)
    else:
        cap = max(1, T * ms)
    tok = np.zeros(cap, np.int32)
    frm = np.zeros(cap, np.int32)
    sc = np.zeros(cap, np.float32)
    du = np.zeros(cap, np.int32)
    dcap = cap + T + 1 if record else 0
    decs = (OrcDecision * max(dcap, 1))()
    nd = C.c_int()
    tot = C.c_double()
    cd = d.to_c()
    n = lib().orc_decode_utt(C.byref(cd), _ptr_array(params), _fp(feats), T, int(out_len),
                             ms, int(tdt), _ip(tok), _ip(frm), _fp(sc), _ip(du), cap,
                             decs if record else None, dcap, C.byref(nd), C.byref(tot))
    h = Hyp(tok[:n].tolist(), frm[:n].tolist(), sc[:n].copy(), tot.value,
            du[:n].tolist() if tdt else [])
    if record:
        h.decisions = [(decs[i].t, decs[i].k, decs[i].margin, decs[i].dur, decs[i].dur_margin)
                       for i in range(min(nd.value, dcap))]
    return h


def decode_batch(d: Dims, params, x, out_len, ms, tdt, record=False):
    return [decode_utt(d, params, x[b], out_len[b], ms, tdt, record) for b in range(x.shape[0])]


def joint(d: Dims, params, f, g_state):
    """run_joint / run_joint_tdt over full state rows (model.cpp:178-213)."""
    f = np.ascontiguousarray(f, np.float32)
    g_state = np.ascontiguousarray(g_state, np.float32)
    B = f.shape[0]
    W = d.state_width
    off = 0 if d.cell == CELL_TANH else 2 * (d.layers - 1) * d.hidden
    logp = np.zeros((B, d.vocab + 1), np.float32)
    D = len(d.durations)
    dl = np.zeros((B, max(D, 1)), np.float32)
    gv = g_state.reshape(-1)[off:]
    gview = np.ascontiguousarray(gv)
    cd = d.to_c()
    lib().orc_joint(C.byref(cd), _ptr_array(params), B, _fp(f), _fp(gview), W, _fp(logp),
                    _fp(dl) if D else None)
    return logp, (dl[:, :D] if D else None)


def prediction(d: Dims, params, labels, state):
    labels = np.ascontiguousarray(labels, np.int32)
    state = np.ascontiguousarray(state, np.float32)
    out = np.zeros_like(state)
    cd = d.to_c()
    lib().orc_prediction(C.byref(cd), _ptr_array(params), labels.shape[0], _ip(labels),
                         _fp(state), _fp(out))
    return out


# ----------------------------------------------------------------- reference
REF_ALGOS = {"oracle": 0, "oracle_tdt": 8, "baseline": 1, "sync_free": 2, "graph_fs": 3,
             "label_loop": 4, "graph_ll": 5, "tdt": 6, "graph_tdt": 7}


def _unpack(counts, tok, frm, sc, tot, cap):
    hyps = []
    for b in range(len(counts)):
        n = int(counts[b])
        hyps.append(Hyp(tok[b, :n].tolist(), frm[b, :n].tolist(), sc[b, :n].copy(), float(tot[b])))
    return hyps


def ref_random_case(seed: int, with_durations: bool, algo: str):
    """Run an unmodified reference decoder on make_random_case(seed)."""
    R = ref()
    cap = 20 * 5 + 1
    cnt = np.zeros(8, np.int32)
    tok = np.zeros((8, cap), np.int32)
    frm = np.zeros((8, cap), np.int32)
    sc = np.zeros((8, cap), np.float32)
    tot = np.zeros(8, np.float64)
    je = C.c_int64()
    B = R.ref_random_case_decode(seed, int(with_durations), REF_ALGOS[algo], _ip(cnt), _ip(tok),
                                 _ip(frm), _fp(sc), tot.ctypes.data_as(C.POINTER(C.c_double)),
                                 cap, C.byref(je))
    if B < 0:
        raise RuntimeError(R.ref_last_error().decode())
    return _unpack(cnt[:B], tok, frm, sc, tot, cap), je.value


def ref_random_case_params(seed: int, with_durations: bool, d: Dims):
    arrs = [np.zeros(s, np.float32) for s in param_shapes(d)]
    ref().ref_random_case_params(seed, int(with_durations), _ptr_array(arrs))
    return arrs


class RefModel:
    """Reference NeuralModel (tanh) or the LstmModel oracle extension."""

    def __init__(self, d: Dims, params):
        self.d = d
        self._params = [np.ascontiguousarray(p, np.float32) for p in params]
        cd = d.to_c()
        self.h = ref().ref_model_create(C.byref(cd), _ptr_array(self._params))
        if not self.h:
            raise RuntimeError(ref().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_model_destroy(self.h)
            self.h = None

    def decode(self, algo: str, x, out_len, ms, threads=1):
        x = np.ascontiguousarray(x, np.float32)
        out_len = np.ascontiguousarray(out_len, np.int32)
        B, T, _ = x.shape
        cap = T * ms + 1
        cnt = np.zeros(B, np.int32)
        tok = np.zeros((B, cap), np.int32)
        frm = np.zeros((B, cap), np.int32)
        sc = np.zeros((B, cap), np.float32)
        tot = np.zeros(B, np.float64)
        secs = C.c_double()
        rc = ref().ref_decode(self.h, REF_ALGOS[algo], _fp(x), B, T, _ip(out_len), ms, threads,
                              _ip(cnt), _ip(tok), _ip(frm), _fp(sc),
                              tot.ctypes.data_as(C.POINTER(C.c_double)), cap, C.byref(secs))
        if rc != 0:
            raise RuntimeError(ref().ref_last_error().decode())
        return _unpack(cnt, tok, frm, sc, tot, cap), secs.value

    def joint(self, f, g_state):
        f = np.ascontiguousarray(f, np.float32)
        g_state = np.ascontiguousarray(g_state, np.float32)
        B = f.shape[0]
        D = len(self.d.durations)
        logp = np.zeros((B, self.d.vocab + 1), np.float32)
        dl = np.zeros((B, max(D, 1)), np.float32)
        ref().ref_joint(self.h, B, _fp(f), _fp(g_state), _fp(logp), _fp(dl) if D else None)
        return logp, (dl[:, :D] if D else None)

    def prediction(self, labels, state):
        labels = np.ascontiguousarray(labels, np.int32)
        state = np.ascontiguousarray(state, np.float32)
        out = np.zeros_like(state)
        ref().ref_prediction(self.h, labels.shape[0], _ip(labels), _fp(state), _fp(out))
        return out


def hyps_equal(a, b) -> bool:
    """Hypothesis::operator== (decoders.hpp:37): bitwise tokens/frames/scores/total."""
    if len(a) != len(b):
        return False
    for x, y in zip(a, b):
        if list(x.tokens) != list(y.tokens) or list(x.frames) != list(y.frames):
            return False
        if np.asarray(x.scores, np.float32).tobytes() != np.asarray(y.scores, np.float32).tobytes():
            return False
        if x.total_score != y.total_score:
            return False
    return True
