#!/usr/bin/env python3
"""Summarise ncu artefacts into profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py launches <launches.csv>            -> per-kernel shares
  python tools/ncu_summary.py report <x.ncu-rep> [alg_bytes]     -> key metrics JSON
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_of_peak",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "smsp__inst_executed.sum": "warp_instructions",
}


def to_bytes(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v.replace(",", "")) * mult.get(unit, 1)


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in data:
        if len(r) > vi:
            agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append({"kernel": k, "launches": len(v), "mean_us": round(sum(v) / len(v) / 1e3, 2),
                    "total_us": round(sum(v) / 1e3, 1), "share": round(sum(v) / tot, 4)})
    return out


def report(path, alg_bytes=None, match=None):
    """Summary of the first launch in the report (or the first whose kernel
    name contains `match`)."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    ki = h.index("Kernel Name")
    v = next(r for r in rows[2:] if match is None or match in r[ki])
    out = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else None}
    for i, n in enumerate(h):
        if n in KEYS:
            val = v[i]
            if u[i] in ("byte", "Kbyte", "Mbyte", "Gbyte"):
                out[KEYS[n]] = to_bytes(val, u[i])
            else:
                try:
                    out[KEYS[n]] = float(val.replace(",", ""))
                except ValueError:
                    out[KEYS[n]] = val
                out[KEYS[n] + "_unit"] = u[i]
    stalls = {n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(v[i] or 0)
              for i, n in enumerate(h) if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("per_issue_active.ratio")}
    out["top_stalls"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:5])
    if "dram_read" in out:
        out["dram_bytes_per_launch"] = out["dram_read"] + out.get("dram_write", 0)
    if alg_bytes:
        out["alg_bytes_per_launch"] = alg_bytes
        out["traffic_over_alg"] = round(out["dram_bytes_per_launch"] / alg_bytes, 4)
    return out


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    else:
        print(json.dumps(report(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] else None,
                                sys.argv[4] if len(sys.argv) > 4 else None), indent=1))
