"""Host-side mirror of the reference decoder interface, backed by the CUDA
library through the C ABI (include/rnntg.h).

Reference: /root/reference/proj/include/rnntsim/decoders.hpp:56-130 and
model.hpp:92-161.  Names, argument meaning and error behaviour follow the
reference; the simulated ``Engine&`` argument has no counterpart here (the
device is real: each CapturedDecoder owns a CUDA stream).

    model = Model(dims, weights)                      # DecoderModel (on device)
    hyps  = greedy_decode_sync_free(model, x, out_len, max_symbols)
    cap   = build_decode_graph(model, DecodeAlgo.LabelLoop, B, T, ms)
    hyps  = replay_decode(cap, x, out_len)
"""
from __future__ import annotations

import ctypes as C
import enum
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import errors
from ._lib import Dims as _CDims
from ._lib import Stats as _CStats
from ._lib import check, lib

CELL = {"tanh": 0, "lstm": 1}


class DecodeAlgo(enum.IntEnum):
    """decoders.hpp:97"""
    FrameSync = 0
    LabelLoop = 1
    TdtLabelLoop = 2


class Exec(enum.IntEnum):
    Graph = 0        # CUDA graph with nested conditional WHILE nodes (tcgen05 step kernel bodies)
    Persistent = 1   # persistent kernel alternative (FFMA, shared-memory weights)
    Tensor = 2       # persistent kernel on tcgen05 tensor cores, role-specialised CTAs
    HostLoop = 3     # sync-requiring baseline: same kernels, host loop with a flag sync per step
    GraphFFMA = 4    # CUDA graph over the FFMA step kernels (4 nodes per inner step)


@dataclass
class ModelDims:
    """RnntDims (model.hpp:31-40) + prediction-network cell and depth."""
    vocab: int
    embed: int
    hidden: int
    joint: int
    feature: int
    durations: tuple = ()
    cell: str = "tanh"
    layers: int = 1

    def to_c(self) -> _CDims:
        d = _CDims(self.vocab, self.embed, self.hidden, self.layers, CELL[self.cell], self.joint,
                   self.feature, len(self.durations))
        for i, v in enumerate(self.durations):
            d.durations[i] = int(v)
        return d

    @property
    def blank_index(self) -> int:
        return self.vocab

    @property
    def state_width(self) -> int:
        return self.hidden if self.cell == "tanh" else 2 * self.layers * self.hidden

    def param_shapes(self):
        from .synth import param_shapes
        return param_shapes(self.vocab, self.embed, self.hidden, self.joint, self.feature,
                            self.durations, self.cell, self.layers)


@dataclass
class Hypothesis:
    """decoders.hpp:31-38, plus the TDT duration of each emission."""
    tokens: list
    frames: list
    scores: np.ndarray
    total_score: float
    durations: list = field(default_factory=list)

    def __eq__(self, other):  # bitwise, like Hypothesis::operator==
        return (list(self.tokens) == list(other.tokens) and list(self.frames) == list(other.frames)
                and np.asarray(self.scores, np.float32).tobytes()
                == np.asarray(other.scores, np.float32).tobytes()
                and self.total_score == other.total_score)


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


class Model:
    """Device-resident DecoderModel (NeuralModel tanh-RNN or stacked LSTM)."""

    def __init__(self, dims: ModelDims, weights, device: int = 0):
        self.dims = dims
        shapes = dims.param_shapes()
        if len(weights) != len(shapes):
            raise errors.ValueError(f"expected {len(shapes)} weight tensors, got {len(weights)}")
        ws = []
        for w, s in zip(weights, shapes):
            a = np.ascontiguousarray(w, dtype=np.float32)
            if a.size != int(np.prod(s)):
                raise errors.DimensionError(f"weight of size {a.size} does not match {s}")
            ws.append(a)
        arr = (C.POINTER(C.c_float) * len(ws))(*[w.ctypes.data_as(C.POINTER(C.c_float)) for w in ws])
        cd = dims.to_c()
        h = C.c_void_p()
        check(lib().rnntg_model_create(device, C.byref(cd), arr, len(ws), C.byref(h)))
        self._h = h
        self.device = device
        self._decoders = {}
        self._live = weakref.WeakSet()  # every CapturedDecoder built on this model

    @classmethod
    def from_seed(cls, dims: ModelDims, seed: int = 1, device: int = 0, blank_bias: float = 0.0):
        from .synth import init_params
        w = init_params(seed, dims.param_shapes())
        if blank_bias:
            w[-2 if dims.durations else -1][:, dims.vocab] += np.float32(blank_bias)
        return cls(dims, w, device)

    @property
    def handle(self):
        return self._h

    def close(self):
        # every decoder built on this model goes first: a decoder must not
        # outlive its model (decoders.hpp:100-113)
        for d in list(self._live):
            d.close()
        self._decoders.clear()
        if self._h:
            lib().rnntg_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # kernel-level entry points (test_model.cpp:224-270 analogues)
    def joint(self, f, g):
        f = np.ascontiguousarray(f, np.float32)
        g = np.ascontiguousarray(g, np.float32)
        B = f.shape[0]
        logp = np.zeros((B, self.dims.vocab + 1), np.float32)
        D = len(self.dims.durations)
        dl = np.zeros((B, max(D, 1)), np.float32)
        check(lib().rnntg_step_joint(self._h, B, _ptr(f), _ptr(g), _ptr(logp),
                                     _ptr(dl) if D else None))
        return logp, (dl[:, :D] if D else None)

    def prediction(self, labels, state):
        labels = np.ascontiguousarray(labels, np.int32)
        state = np.ascontiguousarray(state, np.float32)
        out = np.zeros_like(state)
        check(lib().rnntg_step_prediction(self._h, labels.shape[0], _ptr(labels), _ptr(state),
                                          _ptr(out)))
        return out

    def enc_proj(self, x):
        x = np.ascontiguousarray(x, np.float32).reshape(-1, self.dims.feature)
        out = np.zeros((x.shape[0], self.dims.joint), np.float32)
        check(lib().rnntg_enc_proj(self._h, x.shape[0], _ptr(x), _ptr(out)))
        return out

    def cached_decoder(self, algo, batch, frames, max_symbols, exec=Exec.Graph):
        key = (int(algo), batch, frames, max_symbols, int(exec))
        if key not in self._decoders:
            self._decoders[key] = CapturedDecoder(self, algo, batch, frames, max_symbols, exec)
        return self._decoders[key]


class CapturedDecoder:
    """build_decode_graph's CapturedDecoder (decoders.hpp:100-113): a decode
    program for fixed (algo, batch, max_frames, max_symbols) with static
    device buffers; fresh batches of the same shape are bound and replayed."""

    def __init__(self, model: Model, algo, batch: int, max_frames: int, max_symbols: int,
                 exec=Exec.Graph):
        self.model = model
        self.algo = DecodeAlgo(int(algo))
        self.batch, self.max_frames, self.max_symbols = batch, max_frames, max_symbols
        self.feature_dim = model.dims.feature
        h = C.c_void_p()
        check(lib().rnntg_decoder_create(model.handle, int(self.algo), int(exec), batch, max_frames,
                                         max_symbols, C.byref(h)))
        self._h = h
        self.capacity = lib().rnntg_decoder_capacity(h)
        model._live.add(self)

    def close(self):
        if getattr(self, "_h", None):
            lib().rnntg_decoder_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def bind_inputs(self, x, out_len):
        """bind_decode_inputs / validate_decode_inputs (decoders.cpp:124-142, 202-207)."""
        x = np.asarray(x)
        out_len = np.asarray(out_len)
        if x.ndim != 3 or x.dtype != np.float32:
            raise errors.DimensionError("features must be float32 [batch, frames, features]")
        if x.shape != (self.batch, self.max_frames, self.feature_dim):
            raise errors.DimensionError("feature shape does not match the decode program")
        if out_len.ndim != 1 or out_len.dtype != np.int32 or out_len.shape[0] != self.batch:
            raise errors.DimensionError("out_len must be int32 [batch]")
        self._x = np.ascontiguousarray(x)
        self._len = np.ascontiguousarray(out_len)
        check(lib().rnntg_bind(self._h, _ptr(self._x), _ptr(self._len)))

    def launch(self):
        check(lib().rnntg_launch(self._h))

    def sync(self):
        check(lib().rnntg_sync(self._h))

    def read_hypotheses(self):
        """read_emissions (decoders.cpp:97-122)."""
        B, cap = self.batch, self.capacity
        cnt = np.zeros(B, np.int32)
        tok = np.zeros((B, cap), np.int32)
        frm = np.zeros((B, cap), np.int32)
        sc = np.zeros((B, cap), np.float32)
        du = np.zeros((B, cap), np.int32)
        check(lib().rnntg_read(self._h, _ptr(cnt), _ptr(tok), _ptr(frm), _ptr(sc), _ptr(du), cap))
        out = []
        for b in range(B):
            n = int(cnt[b])
            s = sc[b, :n].copy()
            total = float(np.cumsum(s.astype(np.float64))[-1]) if n else 0.0
            out.append(Hypothesis(tok[b, :n].tolist(), frm[b, :n].tolist(), s, total,
                                  du[b, :n].tolist() if self.algo == DecodeAlgo.TdtLabelLoop else []))
        return out

    def stats(self) -> dict:
        s = _CStats()
        check(lib().rnntg_get_stats(self._h, C.byref(s)))
        return {"joint_evals": s.joint_evals, "pred_steps": s.pred_steps,
                "outer_iters": s.outer_iters, "emitted": s.emitted, "gpu_ms": s.gpu_ms}


def build_decode_graph(model: Model, algo, batch: int, max_frames: int, max_symbols: int,
                       exec=Exec.Graph) -> CapturedDecoder:
    """decoders.cpp:589-627"""
    return CapturedDecoder(model, algo, batch, max_frames, max_symbols, exec)


def replay_decode(captured: CapturedDecoder, x, out_len):
    """decoders.cpp:629-639: bind, one launch, read."""
    if captured is None or not captured.handle:
        raise errors.StateError("captured decoder is not initialized")
    captured.bind_inputs(x, out_len)
    captured.launch()
    return captured.read_hypotheses()


def decode_joint_evals(captured: CapturedDecoder) -> int:
    """decoders.cpp:641-643 (joint-step launches of the last decode)."""
    return captured.stats()["joint_evals"]


def _eager(model: Model, algo, x, out_len, max_symbols, exec=Exec.Graph):
    x = np.asarray(x)
    if x.ndim != 3:
        raise errors.DimensionError("features must be rank 3 [batch, frames, features]")
    if max_symbols < 1:
        raise errors.ValueError("max_symbols must be >= 1")
    dec = model.cached_decoder(algo, x.shape[0], x.shape[1], max_symbols, exec)
    return replay_decode(dec, x, out_len)


def greedy_decode_sync_free(model: Model, x, out_len, max_symbols: int, exec=Exec.Graph):
    """decoders.cpp:565-575 -- frame-looping, no host sync per symbol."""
    return _eager(model, DecodeAlgo.FrameSync, x, out_len, max_symbols, exec)


def label_looping_decode(model: Model, x, out_len, max_symbols: int, exec=Exec.Graph):
    """decoders.cpp:577-580"""
    return _eager(model, DecodeAlgo.LabelLoop, x, out_len, max_symbols, exec)


def tdt_label_looping_decode(model: Model, x, out_len, max_symbols: int, exec=Exec.Graph):
    """decoders.cpp:582-587"""
    if not model.dims.durations:
        raise errors.StateError("duration-head decoding needs a model with a duration head")
    return _eager(model, DecodeAlgo.TdtLabelLoop, x, out_len, max_symbols, exec)
