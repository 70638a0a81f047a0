"""Synthetic weights and encoder outputs, byte-identical to the reference's
generators: splitmix64 ``Rng`` (tensor.cpp:633-653) with the fixed float
mapping lo + (hi - lo) * (u >> 40) * 2^-24, and ``init_params``'s fill order
(model.cpp:81-108; the LSTM layout keeps the order with one (w_ih, w_hh,
bias) triple per layer).  Vectorised with numpy uint64 arithmetic.
"""
from __future__ import annotations

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, n: int, start: int = 0) -> np.ndarray:
    """Draws start..start+n-1 of Rng(seed).next_u64()."""
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, n: int, lo: float, hi: float, start: int = 0) -> np.ndarray:
    u = (splitmix64(seed, n, start) >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)
    lo32, hi32 = np.float32(lo), np.float32(hi)
    return lo32 + (hi32 - lo32) * u


def param_shapes(vocab, embed, hidden, joint, feature, durations=(), cell="tanh", layers=1):
    v1 = vocab + 1
    g = 4 * hidden if cell == "lstm" else hidden
    shapes = [(v1, embed)]
    for l in range(layers):
        shapes += [(embed if l == 0 else hidden, g), (hidden, g), (g,)]
    shapes += [(feature, joint), (hidden, joint), (joint, v1)]
    if durations:
        shapes.append((joint, len(durations)))
    return shapes


def init_params(seed: int, shapes) -> list:
    """init_params: U[-0.08, 0.08) from Rng(seed) in fill order."""
    total = sum(int(np.prod(s)) for s in shapes)
    flat = uniform(seed, total, -0.08, 0.08)
    out, o = [], 0
    for s in shapes:
        n = int(np.prod(s))
        out.append(flat[o:o + n].reshape(s).copy())
        o += n
    return out


def encoder_outputs(seed: int, batch: int, frames: int, feature: int) -> np.ndarray:
    """x ~ U[-1, 1) from Rng(seed), [B,T,F] row-major (decode_test_util.hpp:54)."""
    return uniform(seed, batch * frames * feature, -1.0, 1.0).reshape(batch, frames, feature)
