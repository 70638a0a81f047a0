#!/usr/bin/env python
"""Benchmark: decoded encoder frames/s of the B200 RNN-T greedy decoder.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c3|c4|c5|c1] [--exec tensor|persistent|graph]

A "step" is one decode of one batch through the captured program (K1 encoder
projection + the device-resident decode loops).  Default workload (N=1) is
BASELINE.json configs[1] (C2): Parakeet-RNNT-1.1B-shaped decoder -- encoder
dim 1024, 2-layer LSTM 640, joint 640, V=1025 (1024 + blank), B=32, T=250,
frame-looping, max_symbols=5, fp32, random-init weights (Rng(1)) and synthetic
encoder outputs (Rng(2)).  Under torchrun each rank decodes its own B=32 batch
(weak scaling, no collective on the data path: utterances are independent);
--config c5 splits B=256, T=500 across ranks (strong scaling).

Timing: W untimed warm-up decodes, then K decodes each bracketed by CUDA
events on the decoder stream, with L2 flushed (256 MiB write) before every
timed decode; barrier + synchronize around the timed region; max over ranks.
`e2e` repeats the measurement through the C ABI with host buffers: pinned
host -> device copy of x and out_len, launch, device -> host read of the
emissions, all inside the timed region; by default as a serving pipeline
(step i+1's host -> device copy on a copy stream overlaps step i's decode,
the decoder binds from the device copy), --e2e-serial for the serial form.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (algo, B, T, ms, durations, layers, hidden, joint, vocab, feature, scaling)
    "c1": ("fs", 4, 200, 5, (), 1, 320, 320, 128, 256, "weak"),
    "c2": ("fs", 32, 250, 5, (), 2, 640, 640, 1024, 1024, "weak"),
    "c3": ("ll", 32, 250, 10, (), 2, 640, 640, 1024, 1024, "weak"),
    "c4": ("tdt", 32, 250, 10, (0, 1, 2, 3, 4), 2, 640, 640, 1024, 1024, "weak"),
    "c5": ("fs", 256, 500, 5, (), 2, 640, 640, 1024, 1024, "strong"),
}
ALGO_ID = {"fs": 0, "ll": 1, "tdt": 2}
EXEC_ID = {"graph": 0, "persistent": 1, "tensor": 2, "hostloop": 3, "graph_ffma": 4}
ALGO_NAME = {"fs": "frame-looping", "ll": "label-looping", "tdt": "TDT label-looping"}
METRIC = "decoded encoder frames/sec (Parakeet-1.1B dec, B=32); GPU idle %; µs/step"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--exec", default="tensor", choices=["tensor", "graph", "persistent", "hostloop", "graph_ffma"],
                    help="tensor: persistent kernel on tcgen05 tensor cores (default, fastest; falls "
                         "back to persistent when the shape does not fit it), persistent: FFMA "
                         "persistent kernel, graph: conditional-WHILE CUDA graph, hostloop: the "
                         "sync-requiring baseline (same kernels, host loop with a flag sync per step)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-serial", action="store_true",
                    help="e2e without overlapping the next step's host->device copy with this step's decode")
    ap.add_argument("--no-compare", action="store_true",
                    help="skip timing the other executors")
    ap.add_argument("--blank-bias", type=float, default=0.0)
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="target duration of the bounded CPU reference sample")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def shard(cfg, rank, world):
    algo, B, T, ms, durs, L, H, J, V, F, scaling = cfg
    if scaling == "strong":
        b0, b1 = B * rank // world, B * (rank + 1) // world
    else:
        b0, b1 = B * rank, B * (rank + 1)
    return b0, b1


def make_inputs(cfg, b0, b1):
    from paper_2406_03791_b200 import synth
    algo, B, T, ms, durs, L, H, J, V, F, scaling = cfg
    n = (b1 - b0) * T * F
    x = synth.uniform(2, n, -1.0, 1.0, start=b0 * T * F).reshape(b1 - b0, T, F)
    lens = np.full(b1 - b0, T, np.int32)
    return x, lens


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.proc = None
        self.th = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
            # the first sample arrives ~0.1-0.5 s after the query starts: wait for
            # it so a short timed region is still covered by the 100 ms stream
            t0 = time.time()
            while not self.samples and time.time() - t0 < 5.0:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        self.n_pre = len(self.samples)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.th:
            self.th.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        note = None
        if len(self.samples) > self.n_pre:
            self.samples = self.samples[self.n_pre:]  # the samples taken inside the timed region
        else:  # region shorter than the sampling period: the sample at its start
            self.samples = self.samples[-1:]
            note = "timed region shorter than the 100 ms sampling period: the sample taken as it started"
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for i, n in enumerate(names):
                if s[4 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples), **({"note": note} if note else {})}


def cpu_reference_sample(cfg, seconds_target, threads=None, blank_bias=0.0):
    """The reference's own decoders (oracle/_ref: rnnt-sim compiled from its
    sources + the LstmModel extension) on a bounded sample of the workload."""
    from oracle import oracle as O
    algo, B, T, ms, durs, L, H, J, V, F, scaling = cfg
    d = O.Dims(V, H, H, J, F, durs, O.CELL_LSTM, L)
    p = O.init_params(1, d)
    if blank_bias:
        p[-2 if durs else -1][:, V] += np.float32(blank_bias)
    m = O.RefModel(d, p)
    nproc = os.cpu_count() or 1
    threads = threads or min(nproc, B)
    ref_algo = {"fs": "sync_free", "ll": "label_loop", "tdt": "tdt"}[algo]
    Bs = threads  # one utterance per thread
    # calibrate on 2 frames, then size the sample to ~seconds_target
    x, lens = make_inputs(cfg, 0, Bs)
    Ts = 2
    _, secs = m.decode(ref_algo, np.ascontiguousarray(x[:, :Ts]), np.full(Bs, Ts, np.int32), ms,
                       threads)
    Ts = int(max(2, min(T, Ts * seconds_target / max(secs, 1e-3))))
    _, secs = m.decode(ref_algo, np.ascontiguousarray(x[:, :Ts]), np.full(Bs, Ts, np.int32), ms,
                       threads)
    frames = Bs * Ts
    return {"value": frames / secs, "unit": "frames/s", "cores": threads, "kind": "reference",
            "sample": f"{Bs} utterances x {Ts} frames of {ALGO_NAME[algo]} (ms={ms}), "
                      f"reference rnnt-sim decoders + LstmModel, {threads} threads of {nproc}",
            "seconds": secs}


def prefix_check(cfg, name, hyps, Ts):
    """Reference-arm hypotheses (utterances decoded over their first Ts frames)
    against the full-size fixture: every decoder here is causal in t, so the
    truncated decode equals the full decode's emissions at frames < Ts."""
    from tests.parity import FullsizeFixture
    algo, B, T, ms, durs, L, H, J, V, F, scaling = cfg
    path = os.path.join(ROOT, "tests", "golden", f"fullsize_{name}.npz")
    if not os.path.exists(path):
        return {"checked": False, "why": "no fixture"}
    fx = FullsizeFixture(name)
    if (fx.meta["B"], fx.meta["T"], fx.meta["ms"], fx.meta["algo"]) != (B, T, ms, algo):
        return {"checked": False, "why": "fixture is for another configuration"}
    bad = []
    for b, h in enumerate(hyps):
        t, f, sc, _ = fx.utt(b)
        k = int(np.sum(f < Ts))
        if (list(h.tokens) != t[:k].tolist() or list(h.frames) != f[:k].tolist()
                or np.asarray(h.scores, np.float32).tobytes() != sc[:k].astype(np.float32).tobytes()):
            bad.append(b)
    return {"checked": True, "fixture": f"tests/golden/fullsize_{name}.npz", "utterances": len(hyps),
            "frames_each": Ts, "bitwise_equal": len(hyps) - len(bad), "mismatched": bad}


def run_reference_arm(args, cfg, rank, world):
    """--impl reference: the reference's own batched decoders (oracle/_ref =
    rnnt-sim compiled from /root/reference sources + the LstmModel extension;
    greedy_decode_sync_free / label_looping_decode / tdt_label_looping_decode)
    on the box's host cores, one utterance per thread.  Each step decodes the
    same bounded sample of the workload -- the first min(B, cores) utterances
    of the config over their first Ts frames, Ts sized so the whole
    --warmup + --steps run takes about two minutes -- and is timed on the
    wall clock; the hypotheses are checked bit for bit against the prefix of
    the committed full-size fixture."""
    if rank != 0:
        return
    from oracle import oracle as O
    algo, B, T, ms, durs, L, H, J, V, F, scaling = cfg
    d = O.Dims(V, H, H, J, F, durs, O.CELL_LSTM, L)
    p = O.init_params(1, d)
    if args.blank_bias:
        p[-2 if durs else -1][:, V] += np.float32(args.blank_bias)
    m = O.RefModel(d, p)
    nproc = os.cpu_count() or 1
    threads = min(nproc, B)
    ref_algo = {"fs": "sync_free", "ll": "label_loop", "tdt": "tdt"}[algo]
    x, _ = make_inputs(cfg, 0, threads)
    secs_per_step = max(0.2, min(20.0, args.cpu_seconds, 120.0 / max(args.steps + args.warmup, 1)))
    _, s2 = m.decode(ref_algo, np.ascontiguousarray(x[:, :2]), np.full(threads, 2, np.int32), ms, threads)
    Ts = int(max(2, min(T, 2 * secs_per_step / max(s2, 1e-3))))
    xs = np.ascontiguousarray(x[:, :Ts])
    ls = np.full(threads, Ts, np.int32)
    secs = []
    hyps = None
    for i in range(args.warmup + args.steps):
        hyps, sec = m.decode(ref_algo, xs, ls, ms, threads)
        if i >= args.warmup:
            secs.append(sec)
    sec = float(np.mean(secs)) if secs else sec
    v = threads * Ts / sec
    chk = prefix_check(cfg, args.config + ("b" if args.blank_bias else ""), hyps, Ts)
    sample = (f"{threads} of the {B} utterances x their first {Ts} of {T} frames per step, "
              f"{ALGO_NAME[algo]} (ms={ms}); reference rnnt-sim decoders ({ref_algo}) + LstmModel, "
              f"one utterance per thread, {threads} threads of {nproc}")
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "frames/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1000.0 * sec, "higher_is_better": True,
           "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": config_json(args, cfg) | {"parallelism": f"utterance-sharded x{world}"},
           "cpu_baseline": {"kind": "reference", "cores": threads, "sample": sample, "value": v,
                            "unit": "frames/s"},
           "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "parity": chk}
    print(json.dumps(out), flush=True)


def step_weight_bytes(cfg):
    """Algorithmic fp32 weight bytes of one prediction step and of one joint
    step: every LSTM layer's W_ih and W_hh (layer 0's input
    is the embedding, E = H in every BASELINE config), the biases, pred_proj;
    the joint's out_proj (+ dur_proj).  K6 reads a table0 row per label
    instead of multiplying emb @ W_ih0; the figure follows the reference's
    algorithm.  C2: 27.87 + 2.62 = 30.497 MB per inner step."""
    algo, B, T, ms, durs, L, H, J, V, F, scaling = cfg
    return 4 * (H * 4 * H * 2 * L + 4 * H * L + H * J), 4 * J * (V + 1 + len(durs))


def roofline_block(args, L_, dh, st, cfg, Bl, ms_per_step, clk, persistent, step_ms=None, step_launches=None):
    """Dominant kernel's achieved bandwidth / FLOP rate, measured with CUDA
    events on standalone launches of the decoder's own kernels (step_ms: the
    tcgen05 step kernel's mean launch time from the CUPTI trace, for the graph
    / host-loop executors)."""
    from paper_2406_03791_b200._lib import check
    algo, B, T, ms, durs, L, H, J, V, F, scaling = cfg
    kern = {}
    names = {0: "enc_proj"}
    if persistent:
        names[10] = "persistent"
    elif step_ms is not None:
        kern["ptc_step"] = step_ms
    else:
        names.update({1: "pred_layer0", 2: "pred_layer1", 8: "pred_proj", 9: "joint"})
    for w, n in names.items():
        if w in (1, 2) and w - 1 >= L:
            continue
        ms_ = C.c_float()
        check(L_.rnntg_time_kernel(dh, w, 3 if w == 10 else 20, C.byref(ms_)))
        kern[n] = ms_.value
    Hp = (H + 63) // 64 * 64
    Jp = (J + 63) // 64 * 64
    Bp = (Bl + 31) // 32 * 32
    # the tensor executor decodes up to 256 rows in one kernel as <= 32-row
    # groups (stats count group-steps); beyond 256 as sub-decodes back to back
    n_sub = (Bl + 255) // 256 if (persistent and args.exec == "tensor" and Bl > 256) else 1
    Brow = min(Bl, 32)
    # the stats count group-steps (<= 32 rows each); the weights of a step are
    # read once for all ceil(B / 32) groups (on chip), so per launch the
    # algorithmic weight bytes are those of the batch steps = group-steps / groups
    ngrp = max(1, -(-Bl // 32)) if Bl <= 256 else 8
    V1 = V + 1
    V1p = (V1 + 15) // 16 * 16
    Dn = len(durs)
    pred_w, joint_w = step_weight_bytes(cfg)
    bytes_per = {  # algorithmic bytes per launch (weights + activations read + outputs written)
        "pred_layer1": 4 * (2 * Hp * 4 * Hp + Bp * 2 * Hp + 2 * Bp * Hp * 2),
        "pred_layer0": 4 * (Hp * 4 * Hp + Bp * Hp + 2 * Bp * Hp * 2 + Bp * 4 * Hp),
        "pred_proj": 4 * (Hp * Jp + Bp * Hp + Bp * Jp),
        "joint": 4 * (Jp * V1p + 2 * Bp * Jp),
        "enc_proj": 4 * (Bl * T * F + F * Jp + Bl * T * Jp),
        "persistent": (st.pred_steps * pred_w + st.joint_evals * joint_w) / n_sub / ngrp,
        # (a step launch runs up to RNNTG_GRAPH_STEPS decisions: the decode's
        # bytes over its step launches)
        "ptc_step": (st.pred_steps * pred_w + st.joint_evals * joint_w) / max(step_launches or st.joint_evals, 1),
    }
    pred_f = 2 * Brow * (4 * H * H * 2 * L + H * J)
    joint_f = 2 * Brow * J * (V1 + Dn)
    flops_per = {
        "pred_layer1": 2 * Bl * 2 * H * 4 * H, "pred_layer0": 2 * Bl * H * 4 * H,
        "pred_proj": 2 * Bl * H * J, "joint": 2 * Bl * J * V1, "enc_proj": 2 * Bl * T * F * J,
        "persistent": (st.pred_steps * pred_f + st.joint_evals * joint_f) / n_sub,
        "ptc_step": (st.pred_steps * pred_f + st.joint_evals * joint_f) / max(step_launches or st.joint_evals, 1),
    }
    per_step_counts = {"enc_proj": 1, "pred_layer0": st.pred_steps,
                       "pred_layer1": st.pred_steps if L > 1 else 0,
                       "pred_proj": st.pred_steps, "joint": st.joint_evals, "persistent": n_sub,
                       "ptc_step": step_launches or st.joint_evals}
    share = {n: kern[n] * per_step_counts[n] / ms_per_step for n in kern}
    dom = max(share, key=share.get)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    clk = clk.summary() if hasattr(clk, "summary") else clk
    sm_mhz = clk.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    fp32_peak = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12
    ach = bytes_per[dom] / (kern[dom] / 1000.0) / 1e9
    fp32_ach = flops_per[dom] / (kern[dom] / 1000.0) / 1e12
    # per inner step roofline (north star): max(weight bytes / HBM, FLOPs / FP32 peak)
    steps = max(st.joint_evals, 1)
    step_bytes = (st.pred_steps * pred_w + st.joint_evals * joint_w) / steps / ngrp  # (weights shared by the groups)
    step_flops = (st.pred_steps * pred_f + st.joint_evals * joint_f) / steps
    t_step = ms_per_step * 1000.0 / steps
    tensor = args.exec in ("tensor", "graph", "hostloop")
    tc_peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1378.6)))
    # tensor executor: the fp32 GEMVs run as 3 fp16 tcgen05 products (hi.hi, hi.lo,
    # lo.hi), so the compute bound is 3x the FLOPs at the dense fp16 tensor peak;
    # the FFMA executors are bound by the FP32 CUDA-core peak
    t_flops = step_flops * 3 / (tc_peak * 1e6) if tensor else step_flops / (fp32_peak * 1e6)
    t_roof = max(step_bytes / (hbm_peak * 1e3), t_flops)
    kname = {"persistent": "ptc_kernel" if tensor else "persistent_kernel",
             "ptc_step": "ptc_kernel (step launches)"}.get(dom, dom)
    extra = {}
    traffic = None
    tsrc = next((f for f in ("r2_ncu_tensor_summary.json", "r1_ncu_tensor_summary.json")
                 if os.path.exists(os.path.join(ROOT, "profiles", f))), None)
    try:  # dram read+write bytes per launch from the committed ncu --set full capture
        for e in json.load(open(os.path.join(ROOT, "profiles", tsrc))):
            if args.exec == "tensor" and "ptc_kernel" in e.get("kernel", "") and Bl == 32 and T == 250:
                mb = lambda k: float(e[k].split()[0]) * {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9}[e[k].split()[1]]
                traffic = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
    except Exception:
        traffic = None
    if tensor and dom in ("persistent", "ptc_step"):
        tc_ach = 3 * flops_per[dom] / (kern[dom] / 1000.0) / 1e12
        extra["tensor"] = {"achieved_tflops": tc_ach, "peak_tflops": tc_peak, "frac": tc_ach / tc_peak,
                           "note": "3 fp16 tcgen05 products per fp32 MAC (hi/lo split) vs "
                                   "MEASURED_PEAKS bf16_tflops_sustained; weights resident in "
                                   "smem/TMEM, so the hbm line is the equivalent streaming rate"}
    return {"bound": "hbm", "kernel": kname, "achieved": ach, "peak": hbm_peak, "unit": "GB/s", **extra,
            "frac": ach / hbm_peak, "traffic": traffic,
            "traffic_source": f"profiles/{tsrc} (ncu --set full, C2)" if traffic else None,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)",
            "algorithmic_bytes_per_launch": bytes_per[dom],
            "algorithmic_bytes_source": "SURVEY.md 8(d) weight bytes per prediction / joint step "
                                        "(C2: 30.497 MB per inner step) x the launch's steps",
            "avg_launch_us": kern[dom] * 1000.0,
            "launches_per_step": per_step_counts[dom],
            "fp32": {"achieved_tflops": fp32_ach, "peak_tflops": fp32_peak,
                     "frac": fp32_ach / fp32_peak,
                     "note": "FFMA peak = 148 SM x 128 lanes x 2 x median SM clock under load"},
            "per_step": {"weight_bytes": step_bytes, "flops": step_flops,
                         "roofline_us": t_roof, "measured_us": t_step, "frac": t_roof / t_step},
            "kernel_us": {n: v * 1000.0 for n, v in kern.items()},
            "step_share": share}, clk


def measure_alt_exec(args, L_, model, cfg, xd, ld, Bl, T, frames_all):
    """Time the other executors on the same inputs (graph_k1: the graph with
    one decision per kernel-node launch, RNNTG_GRAPH_STEPS=1)."""
    out = []
    for other in ("tensor", "persistent", "graph", "graph_k1", "graph_ffma", "hostloop"):
        if other == args.exec:
            continue
        if other == "graph_k1":
            os.environ["RNNTG_GRAPH_STEPS"] = "1"
            try:
                r = measure_exec("graph", L_, model, cfg, xd, ld, Bl, T, frames_all)
            finally:
                os.environ.pop("RNNTG_GRAPH_STEPS", None)
            r["exec"] = "graph_k1"
            out.append(r)
        else:
            out.append(measure_exec(other, L_, model, cfg, xd, ld, Bl, T, frames_all))
    return out


def measure_exec(other, L_, model, cfg, xd, ld, Bl, T, frames_all):
    from paper_2406_03791_b200._lib import Stats, check
    algo = cfg[0]
    dh = C.c_void_p()
    rc = L_.rnntg_decoder_create(model.handle, ALGO_ID[algo], EXEC_ID[other], Bl, T,
                                 cfg[3], C.byref(dh))
    if rc != 0:
        return {"exec": other, "unavailable": L_.rnntg_last_error().decode()}
    check(L_.rnntg_bind_device(dh, C.c_void_p(xd.data_ptr()), C.c_void_p(ld.data_ptr())))
    for _ in range(2):
        check(L_.rnntg_launch(dh))
    check(L_.rnntg_sync(dh))
    n = 3
    tot = 0.0
    for _ in range(n):
        check(L_.rnntg_launch(dh))
        check(L_.rnntg_sync(dh))
        s = Stats()
        check(L_.rnntg_get_stats(dh, C.byref(s)))
        tot += s.gpu_ms
    idle = measure_idle(L_, dh, tot / n)
    check(L_.rnntg_decoder_destroy(dh))
    ms = tot / n
    return {"exec": other, "value": frames_all / (ms / 1000.0), "ms_per_step": ms,
            "us_per_step": 1000.0 * ms / max(s.joint_evals, 1), "gpu_idle": idle}


def measure_idle(L_, dh, decode_ms=None):
    """One decode traced with CUPTI kernel activity.  idle_pct = 1 - (union of
    kernel intervals) / (the untraced, event-timed decode time); tracing
    inflates launch gaps, so the traced span is reported separately."""
    from paper_2406_03791_b200._lib import check
    busy, span, nk = C.c_double(), C.c_double(), C.c_int64()
    # one warm-up trace: the first CUPTI session of a process misses the kernels
    # launched from conditional-node bodies of a graph
    if L_.rnntg_trace_begin() != 0:
        return None
    check(L_.rnntg_launch(dh))
    check(L_.rnntg_sync(dh))
    check(L_.rnntg_trace_end(C.byref(busy), C.byref(span), C.byref(nk)))
    if L_.rnntg_trace_begin() != 0:
        return None
    check(L_.rnntg_launch(dh))
    check(L_.rnntg_sync(dh))
    check(L_.rnntg_trace_end(C.byref(busy), C.byref(span), C.byref(nk)))
    if span.value <= 0:
        return None
    ref_ms = decode_ms if decode_ms else span.value
    return {"idle_pct": max(0.0, 100.0 * (1.0 - busy.value / ref_ms)), "busy_ms": busy.value,
            "decode_ms_untraced": decode_ms, "traced_span_ms": span.value,
            "traced_span_idle_pct": 100.0 * (1.0 - busy.value / span.value), "kernels": nk.value,
            "note": "CUPTI kernel records; a persistent kernel's barrier spin counts as busy"}


def read_hyps(L_, dh, Bl):
    """rnntg_read of the last decode -> per-utterance (tokens, frames, scores, durations)."""
    from types import SimpleNamespace
    from paper_2406_03791_b200._lib import check
    cap = L_.rnntg_decoder_capacity(dh)
    cnt = np.zeros(Bl, np.int32)
    arr = [np.zeros((Bl, cap), np.int32) for _ in range(2)] + [np.zeros((Bl, cap), np.float32),
                                                             np.zeros((Bl, cap), np.int32)]
    check(L_.rnntg_read(dh, *[C.c_void_p(a.ctypes.data) for a in [cnt] + arr], cap))
    return [SimpleNamespace(tokens=arr[0][b, :cnt[b]], frames=arr[1][b, :cnt[b]], scores=arr[2][b, :cnt[b]],
                            durations=arr[3][b, :cnt[b]]) for b in range(Bl)]


def check_parity(args, cfg, hyps, b0, b1, rank, world, dist):
    """The timed decode's hypotheses against the committed full-size fixture of
    the reference's scalar oracle (tests/golden/fullsize_*.npz, same inputs):
    tokens / frames / durations exact, scores within 1e-4, near-ties counted."""
    algo, B, T, ms, durs, L, H, J, V, F, scaling = cfg
    name = args.config + ("b" if args.blank_bias else "")
    res = {"fixture": f"tests/golden/fullsize_{name}.npz", "checked": False}
    path = os.path.join(ROOT, res["fixture"])
    try:
        from tests.parity import FullsizeFixture, compare_fullsize
        fx = FullsizeFixture(name) if os.path.exists(path) else None
        if fx is None:
            res["why"] = "no fixture"
        elif (fx.meta["B"], fx.meta["T"], fx.meta["ms"], fx.meta["algo"]) != (B, T, ms, algo) or \
                abs(fx.meta["blank_bias"] - args.blank_bias) > 1e-12:
            res["why"] = "fixture is for another configuration"
        elif b1 > fx.meta["B"]:
            res["why"] = f"rows {b0}..{b1 - 1} are outside the fixture (weak scaling: rank > 0)"
        else:
            sub = FullsizeFixture.__new__(FullsizeFixture)
            sub.__dict__.update(fx.__dict__)
            sub.counts = fx.counts[b0:b1]
            sub.off = fx.off[b0:b1 + 1]
            sub.wins = {(b - b0, i): m for (b, i), m in fx.wins.items() if b0 <= b < b1}
            rep = compare_fullsize(hyps, sub, name)
            res.update(checked=True, utterances=rep.utterances, exact=rep.exact,
                       permitted_near_ties=rep.permitted, failures=len(rep.failures),
                       first_failures=rep.failures[:3], max_score_rel=rep.max_score_rel)
    except Exception as e:  # reported, never silently passed
        res["error"] = repr(e)
    if dist:
        allr = [None] * world
        dist.all_gather_object(allr, res)
        chk = [r for r in allr if r.get("checked")]
        res = {"fixture": res["fixture"], "checked": bool(chk), "ranks_checked": len(chk),
               "utterances": sum(r["utterances"] for r in chk), "exact": sum(r["exact"] for r in chk),
               "permitted_near_ties": sum(r["permitted_near_ties"] for r in chk),
               "failures": sum(r["failures"] for r in chk),
               "max_score_rel": max([r["max_score_rel"] for r in chk], default=None),
               "per_rank": allr}
    if res.get("failures"):
        print(f"bench.py: PARITY FAILURE {res}", file=sys.stderr)
    return res


def config_json(args, cfg):
    algo, B, T, ms, durs, L, H, J, V, F, scaling = cfg
    return {"workload": f"{args.config}: Parakeet-1.1B-shaped {ALGO_NAME[algo]} decode "
                        f"(enc {F}, {L}-layer LSTM {H}, joint {J}, V={V + 1}"
                        f"{', durations ' + str(list(durs)) if durs else ''})",
            "batch": B, "frames": T, "max_symbols": ms, "algo": algo, "exec": args.exec,
            "sharding": f"{scaling}: utterances split across {args.gpus} GPU(s), no collective",
            "weights": "random init Rng(1) U[-0.08,0.08)", "inputs": "Rng(2) U[-1,1), out_len=T",
            "l2": "flushed (256 MiB write) before every timed decode",
            "blank_bias": args.blank_bias}


def spawn_ranks(args):
    """`bench.py --gpus N` without a launcher: re-run this script under
    torch.distributed.run with N ranks on 127.0.0.1 (one process per GPU)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(spawn_ranks(args))
    rank, world, local = dist_env()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, cfg, rank, world)
        return
    import torch
    from paper_2406_03791_b200 import Model, ModelDims
    from paper_2406_03791_b200._lib import Stats, check, lib

    algo, B, T, ms, durs, L, H, J, V, F, scaling = cfg
    # RNNTG_BENCH_SHARE_GPU=1 maps ranks onto the visible GPUs modulo their
    # count (functional check of the N>1 path on a 1-GPU box; gloo plumbing)
    share = os.environ.get("RNNTG_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dist = None
    coll_dev = "cpu"
    if world > 1:
        # no NCCL: shards are independent; gloo carries only the
        # barriers and the max-over-ranks of the device-timed region
        import torch.distributed as dist
        dist.init_process_group("gloo")
    b0, b1 = shard(cfg, rank, world)
    Bl = b1 - b0
    dims = ModelDims(V, H, H, J, F, durs, "lstm", L)
    model = Model.from_seed(dims, 1, device=local, blank_bias=args.blank_bias)
    L_ = lib()
    # CUPTI first: kernels in the conditional bodies of a graph instantiated
    # before the first activity session are missing from its records
    _b, _s, _n = C.c_double(), C.c_double(), C.c_int64()
    if L_.rnntg_trace_begin() == 0:
        L_.rnntg_trace_end(C.byref(_b), C.byref(_s), C.byref(_n))
    dh = C.c_void_p()
    rc = L_.rnntg_decoder_create(model.handle, ALGO_ID[algo], EXEC_ID[args.exec], Bl, T, ms,
                                 C.byref(dh))
    if rc != 0 and args.exec == "tensor":  # shape outside the tensor executor: FFMA persistent
        print(f"tensor executor unavailable ({L_.rnntg_last_error().decode()}); using persistent",
              file=sys.stderr)
        args.exec = "persistent"
        rc = L_.rnntg_decoder_create(model.handle, ALGO_ID[algo], EXEC_ID[args.exec], Bl, T, ms,
                                     C.byref(dh))
    check(rc)
    x, lens = make_inputs(cfg, b0, b1)
    xd = torch.from_numpy(x).cuda()
    ld = torch.from_numpy(lens).cuda()
    check(L_.rnntg_bind_device(dh, C.c_void_p(xd.data_ptr()), C.c_void_p(ld.data_ptr())))
    stream = torch.cuda.ExternalStream(L_.rnntg_decoder_stream(dh), device=local)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def decode_once():
        check(L_.rnntg_launch(dh))

    for _ in range(args.warmup):
        decode_once()
    check(L_.rnntg_sync(dh))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(float(i))
                evs[i][0].record(stream)
            decode_once()
            with torch.cuda.stream(stream):
                evs[i][1].record(stream)
        check(L_.rnntg_sync(dh))
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = float(sum(step_ms))
    if dist:
        t = torch.tensor([total_ms], device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    st = Stats()
    check(L_.rnntg_get_stats(dh, C.byref(st)))
    frames_all = B * T if scaling == "strong" else B * T * world
    value = frames_all * args.steps / (total_ms / 1000.0)
    ms_per_step = total_ms / args.steps
    per_rank_frames = Bl * T
    fs = algo == "fs"
    persistent = args.exec in ("persistent", "tensor")
    # graph / host loop: the tcgen05 step kernel, one launch per decision
    tc_steps = args.exec in ("graph", "hostloop")
    if persistent:
        launches_per_step = 2
    elif tc_steps:  # K1 + P0 + one launch per (up to RNNTG_GRAPH_STEPS) decisions
        k = int(os.environ.get("RNNTG_GRAPH_STEPS", "16")) if args.exec == "graph" else 1
        launches_per_step = 2 + -(-st.joint_evals // max(k, 1))
    else:
        launches_per_step = 2 + st.pred_steps * (L + 1) + st.joint_evals + (st.outer_iters if fs else 0)
    hyps_dev = read_hyps(L_, dh, Bl)  # the timed decodes' hypotheses (device-resident inputs)
    idle = measure_idle(L_, dh, ms_per_step)
    step_ms = step_launches = None
    if tc_steps and idle and idle.get("kernels", 0) > 2:
        step_ms = (idle["busy_ms"] - 0.0) / idle["kernels"]
        step_launches = idle["kernels"] - 2  # (K1 and the P0 launch are the other two)
    roofline, clk = roofline_block(args, L_, dh, st, cfg, Bl, ms_per_step, clk, persistent, step_ms, step_launches)

    # ---- e2e through the C ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        cap = L_.rnntg_decoder_capacity(dh)
        xh = torch.from_numpy(x).pin_memory()
        lh = torch.from_numpy(lens).pin_memory()
        outs = [torch.empty((Bl,), dtype=torch.int32).pin_memory()] + \
               [torch.empty((Bl, cap), dtype=torch.int32).pin_memory() for _ in range(4)]
        ptr = [C.c_void_p(o.data_ptr()) for o in outs]

        def e2e_once():
            check(L_.rnntg_bind(dh, C.c_void_p(xh.data_ptr()), C.c_void_p(lh.data_ptr())))
            check(L_.rnntg_launch(dh))
            check(L_.rnntg_read(dh, ptr[0], ptr[1], ptr[2], ptr[3], ptr[4], cap))

        # pipelined serving loop: step i+1's pinned host -> device copy runs on
        # a copy stream while step i decodes; the decoder binds from the device
        # copy (rnntg_bind_device) once the copy's event has fired
        cs = torch.cuda.Stream(device=local)
        dstream = torch.cuda.ExternalStream(L_.rnntg_decoder_stream(dh), device=local)
        xs = [torch.empty(x.shape, dtype=torch.float32, device=local) for _ in range(2)]
        ls = [torch.empty(lens.shape, dtype=torch.int32, device=local) for _ in range(2)]
        evs = [torch.cuda.Event() for _ in range(2)]

        def h2d(j):
            with torch.cuda.stream(cs):
                xs[j].copy_(xh, non_blocking=True)
                ls[j].copy_(lh, non_blocking=True)
                evs[j].record(cs)

        def e2e_run(n):
            h2d(0)
            for i in range(n):
                j = i & 1
                dstream.wait_event(evs[j])
                check(L_.rnntg_bind_device(dh, C.c_void_p(xs[j].data_ptr()), C.c_void_p(ls[j].data_ptr())))
                check(L_.rnntg_launch(dh))
                if i + 1 < n:
                    h2d(j ^ 1)
                check(L_.rnntg_read(dh, ptr[0], ptr[1], ptr[2], ptr[3], ptr[4], cap))
            torch.cuda.synchronize(local)

        serial = args.e2e_serial
        if serial:
            for _ in range(2):
                e2e_once()
        else:
            e2e_run(2)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        if serial:
            for _ in range(args.steps):
                e2e_once()
        else:
            e2e_run(args.steps)
        el = time.perf_counter() - t0
        if dist:
            t = torch.tensor([el], device=coll_dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": frames_all * args.steps / el, "unit": "frames/s",
               "h2d_bytes_per_step": int(x.nbytes + lens.nbytes),
               "d2h_bytes_per_step": int(4 * Bl + 4 * 4 * Bl * cap),
               "mode": "serial" if serial else
               "pipelined: step i+1's pinned H2D on a copy stream overlaps step i's decode (first copy not overlapped)"}
        # the pipelined / serial e2e path must decode exactly what the
        # device-input decode did (same inputs): counts, tokens, frames, scores
        cnt_h = outs[0].numpy()
        tok_h, frm_h, durs_h = outs[1].numpy(), outs[2].numpy(), outs[4].numpy()
        sc_h = outs[3].numpy().view(np.float32)
        bad = [b for b, h in enumerate(hyps_dev)
               if cnt_h[b] != len(h.tokens) or not np.array_equal(tok_h[b, :cnt_h[b]], h.tokens)
               or not np.array_equal(frm_h[b, :cnt_h[b]], h.frames)
               or sc_h[b, :cnt_h[b]].tobytes() != np.asarray(h.scores, np.float32).tobytes()
               or not np.array_equal(durs_h[b, :cnt_h[b]], h.durations)]
        e2e["matches_device_decode"] = not bad
        if bad:
            print(f"bench.py: e2e hypotheses differ from the device-input decode on rows {bad[:8]}",
                  file=sys.stderr)

    parity = check_parity(args, cfg, hyps_dev, b0, b1, rank, world, dist)
    alt = None
    if not args.no_compare:
        alt = measure_alt_exec(args, L_, model, cfg, xd, ld, Bl, T, frames_all)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import oracle as O
            if O.ref_available():
                cpu = cpu_reference_sample(cfg, args.cpu_seconds, blank_bias=args.blank_bias)
                cpu.pop("seconds", None)
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "error": str(e)}

    if rank == 0:
        inner = st.joint_evals
        out = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "f32 (tensor exec: each fp32 product as 3 fp16 hi/lo tcgen05 products, fp32 accumulate)"
                     if args.exec == "tensor" else "f32",
            "data": "synthetic (random-init weights, random encoder outputs)",
            "config": config_json(args, cfg) | {"parallelism": f"utterance-sharded x{world}"},
            "us_per_step": 1000.0 * ms_per_step / max(inner, 1),
            "inner_steps_per_decode": inner, "pred_steps_per_decode": st.pred_steps,
            "outer_iters_per_decode": st.outer_iters,
            "tokens_per_frame": st.emitted / max(per_rank_frames, 1),
            "gpu_idle_pct": idle["idle_pct"] if idle else None, "gpu_idle": idle,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches_per_step * args.steps),
            "parity": parity,
            "clocks": clk, "step_ms": step_ms, "alt_exec": alt,
        }
        print(json.dumps(out), flush=True)
    check(L_.rnntg_decoder_destroy(dh))
    model.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
