"""Parity comparator between the CUDA decoder and the CPU oracle.

Rule (north star / SURVEY.md §8c): token, frame and duration sequences must
be identical; a divergence is permitted only where the oracle's top-2 margin
(token logp, or duration logp for TDT) at the diverging decision is below
EPS_MARGIN, and such divergences are counted and reported.  Scores (logp of
the emitted label) must agree within RTOL relative, denominator
max(|ref|, 1e-3).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

EPS_MARGIN = 1e-4
RTOL = 1e-4


@dataclass
class ParityReport:
    utterances: int = 0
    exact: int = 0
    permitted: int = 0
    failures: list = field(default_factory=list)
    max_score_rel: float = 0.0

    def merge(self, o: "ParityReport"):
        self.utterances += o.utterances
        self.exact += o.exact
        self.permitted += o.permitted
        self.failures += o.failures
        self.max_score_rel = max(self.max_score_rel, o.max_score_rel)

    @property
    def ok(self):
        return not self.failures


def _score_rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-3)))


def compare_utt(gpu, ref, tdt: bool, tag="") -> ParityReport:
    """gpu: Hypothesis (package); ref: oracle Hyp with decisions recorded."""
    rep = ParityReport(utterances=1)
    gt, rt = list(gpu.tokens), list(ref.tokens)
    gf, rf = list(gpu.frames), list(ref.frames)
    gd = list(gpu.durations) if tdt else []
    rd = list(ref.durations) if tdt else []
    same = gt == rt and gf == rf and (not tdt or gd == rd)
    if same:
        rel = _score_rel(gpu.scores, ref.scores)
        rep.max_score_rel = rel
        if rel > RTOL:
            rep.failures.append(f"{tag}: score rel err {rel:.3g}")
        else:
            rep.exact = 1
        return rep
    # first diverging emission
    n = min(len(gt), len(rt))
    i = next((j for j in range(n) if gt[j] != rt[j] or gf[j] != rf[j]
              or (tdt and gd[j] != rd[j])), n)
    rel = _score_rel(gpu.scores[:i], ref.scores[:i])
    rep.max_score_rel = rel
    # oracle decisions between emission i-1 (exclusive) and emission i (inclusive)
    emit_idx = [k for k, d in enumerate(ref.decisions) if d[1] != ref_blank(ref)]
    lo = emit_idx[i - 1] + 1 if i >= 1 and i - 1 < len(emit_idx) else 0
    hi = emit_idx[i] + 1 if i < len(emit_idx) else len(ref.decisions)
    window = ref.decisions[lo:hi] or ref.decisions[lo:lo + 1]
    margins = [d[2] for d in window] + ([d[4] for d in window] if tdt else [])
    mmin = min(margins) if margins else float("inf")
    if mmin < EPS_MARGIN and rel <= RTOL:
        rep.permitted = 1
    else:
        rep.failures.append(f"{tag}: diverged at emission {i} (oracle margin {mmin:.3g}, "
                            f"score rel {rel:.3g})")
    return rep


_BLANK = {}


def ref_blank(ref):
    return _BLANK.get(id(ref), -1)


def compare_batch(gpu_hyps, ref_hyps, blank: int, tdt: bool, tag="") -> ParityReport:
    rep = ParityReport()
    for b, (g, r) in enumerate(zip(gpu_hyps, ref_hyps)):
        _BLANK[id(r)] = blank
        rep.merge(compare_utt(g, r, tdt, f"{tag}[{b}]"))
        _BLANK.pop(id(r), None)
    if len(gpu_hyps) != len(ref_hyps):
        rep.failures.append(f"{tag}: batch size {len(gpu_hyps)} != {len(ref_hyps)}")
    return rep


def rel_err(a, b, floor=1e-3):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor)))


# ------------------------------------------------------------ full-size fixtures
class FullsizeFixture:
    """tests/golden/fullsize_<name>.npz (tests/golden/make_fullsize.py): the
    reference's scalar oracle (decoders.cpp:670-755) on bench.py's inputs."""

    def __init__(self, name: str):
        import json
        import os
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", f"fullsize_{name}.npz")
        z = np.load(path)
        self.name = name
        self.meta = json.loads(bytes(z["meta"]).decode())
        self.counts = z["counts"].astype(np.int64)
        self.off = np.concatenate([[0], np.cumsum(self.counts)])
        self.tokens = z["tokens"].astype(np.int32)
        self.frames = z["frames"].astype(np.int32)
        self.scores = z["scores"].view(np.float32)
        self.totals = z["totals"]
        self.durations = z["durations"].astype(np.int32) if "durations" in z.files else None
        self.wins = {}
        for b, i, m in z["wins"]:
            self.wins[(int(b), int(i))] = float(m)

    @property
    def tdt(self):
        return self.durations is not None

    def utt(self, b):
        s = slice(self.off[b], self.off[b + 1])
        return (self.tokens[s], self.frames[s], self.scores[s],
                self.durations[s] if self.tdt else None)

    def window_margin(self, b, i):
        """min oracle top-2 margin over the decisions (emission i-1, emission i]
        (windows >= 1e-3 are not stored: they count as 'not a near tie')."""
        return self.wins.get((b, i), np.inf)


def compare_fullsize(gpu_hyps, fx: FullsizeFixture, tag="") -> ParityReport:
    """Same rule as compare_utt, against a full-size fixture."""
    rep = ParityReport()
    if len(gpu_hyps) != len(fx.counts):
        rep.failures.append(f"{tag}: batch size {len(gpu_hyps)} != {len(fx.counts)}")
        return rep
    for b, g in enumerate(gpu_hyps):
        rep.utterances += 1
        rt, rf, rs, rd = fx.utt(b)
        gt = np.asarray(g.tokens, np.int32)
        gf = np.asarray(g.frames, np.int32)
        gd = np.asarray(g.durations, np.int32) if fx.tdt else None
        same = (len(gt) == len(rt) and np.array_equal(gt, rt) and np.array_equal(gf, rf)
                and (not fx.tdt or np.array_equal(gd, rd)))
        if same:
            rel = _score_rel(g.scores, rs)
            rep.max_score_rel = max(rep.max_score_rel, rel)
            if rel > RTOL:
                rep.failures.append(f"{tag}[{b}]: score rel err {rel:.3g}")
            else:
                rep.exact += 1
            continue
        n = min(len(gt), len(rt))
        neq = (gt[:n] != rt[:n]) | (gf[:n] != rf[:n])
        if fx.tdt:
            neq |= gd[:n] != rd[:n]
        i = int(np.argmax(neq)) if neq.any() else n
        rel = _score_rel(np.asarray(g.scores)[:i], rs[:i])
        rep.max_score_rel = max(rep.max_score_rel, rel)
        m = fx.window_margin(b, i)
        if m < EPS_MARGIN and rel <= RTOL:
            rep.permitted += 1
        else:
            rep.failures.append(f"{tag}[{b}]: diverged at emission {i} of {len(rt)} "
                                f"(oracle margin {m:.3g}, score rel {rel:.3g})")
    return rep
