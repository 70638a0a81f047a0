"""Summarise an ncu --set full report into profiles/*.json.

usage: python scripts/ncu_summary.py gpurun_out/ncu_tc_r1g.ncu-rep profiles/r1_ncu_tensor_summary.json

One object per captured launch (last launch per kernel name wins): duration,
DRAM bytes, tensor-pipe activity, occupancy, clocks, launch shape and the
warp-stall sample histogram (smsp__pcsamp_warps_issue_stalled_*).
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "smsp__inst_executed.sum",
]
STALL = "smsp__pcsamp_warps_issue_stalled_"


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    by_kernel = {}
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        e = {"kernel": d.get("Kernel Name", "?")}
        for k in KEYS:
            if k in d:
                e[k] = f"{d[k]} {u.get(k, '')}".strip()
        st = {}
        for k, v in d.items():
            if k.startswith(STALL) and not k.endswith("_not_issued") and v not in ("", "0"):
                st[k[len(STALL):]] = f"{v} {u.get(k, '')}".strip()
        e["stall_samples"] = st
        by_kernel[e["kernel"]] = e
    with open(out, "w") as f:
        json.dump(list(by_kernel.values()), f, indent=1)
    print(f"wrote {out}: {len(by_kernel)} kernel(s)")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
