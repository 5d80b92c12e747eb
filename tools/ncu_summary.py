"""Summarise an ncu capture of the scan kernel into profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep --tag r01_scan_vN \
        --samples 32000000 [--write-const]

Writes profiles/<tag>_summary.json (selected raw metrics + derived per-sample
figures) and, with --write-const, profiles/scan_inst_per_sample.json, the
per-present-pair thread-instruction count and DRAM traffic per pair that
bench.py uses for the ALU roofline (achieved = inst/pair x pairs / live time).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    "gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__thread_inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
]


def read_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kern = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        kern.append({h: (d[h], units[i]) for i, h in enumerate(hdr)})
    return kern


def to_float(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--samples", type=float, required=True, help="present pairs in the profiled launch")
    ap.add_argument("--write-const", action="store_true")
    a = ap.parse_args()
    kern = read_raw(a.rep)[0]
    sel = {}
    for k in KEYS:
        for h, (v, u) in kern.items():
            if h == k:
                sel[k] = {"value": v, "unit": u}
    stalls = {h: v for h, (v, u) in kern.items() if "average_warps_issue_stalled" in h and h.endswith("ratio")
              and (to_float(v) or 0) > 0.1}
    inst = to_float(sel["smsp__inst_executed.sum"]["value"])
    if "smsp__thread_inst_executed.sum" in sel:
        t_inst = to_float(sel["smsp__thread_inst_executed.sum"]["value"])
    else:   # the full set has the per-instruction thread ratio instead
        t_inst = inst * to_float(sel["smsp__thread_inst_executed_per_inst_executed.ratio"]["value"])
    dur_unit = sel["gpu__time_duration.sum"]["unit"]
    dur = to_float(sel["gpu__time_duration.sum"]["value"]) * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}[dur_unit]
    def bytes_of(k):
        v, u = to_float(sel[k]["value"]), sel[k]["unit"]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    dram = bytes_of("dram__bytes_read.sum") + bytes_of("dram__bytes_write.sum")
    derived = {
        "kernel": kern.get("Kernel Name", ("?", ""))[0],
        "duration_s": dur,
        "present_pairs": a.samples,
        "thread_inst_per_pair": t_inst / a.samples,
        "warp_inst_per_pair": to_float(sel["smsp__inst_executed.sum"]["value"]) / a.samples,
        "dram_bytes": dram,
        "dram_bytes_per_pair": dram / a.samples,
        "lane_inst_per_s": t_inst / dur,
    }
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{a.tag}_summary.json"), "w") as f:
        json.dump({"source": os.path.basename(a.rep), "metrics": sel, "stalls": stalls, "derived": derived}, f,
                  indent=1)
    if a.write_const:
        with open(os.path.join(ROOT, "profiles", "scan_inst_per_sample.json"), "w") as f:
            json.dump({"thread_inst_per_sample": derived["thread_inst_per_pair"],
                       "dram_bytes_per_sample": derived["dram_bytes_per_pair"],
                       "source": f"profiles/{a.tag}_summary.json ({os.path.basename(a.rep)})",
                       "note": "per present (occurrence, slot) pair, ncu --set full, one launch"}, f, indent=1)
    print(json.dumps(derived, indent=1))


if __name__ == "__main__":
    main()
