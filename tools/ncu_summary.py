"""Summarise an ncu capture of the split scan kernels into profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep --tag r01_split_vN \
        --pairs 31999955 --occurrences 100000000 [--write-const]

For every kernel launch in the report writes profiles/<tag>_<kernel>.json
(selected raw metrics, stall reasons, derived per-unit figures).  With
--write-const, profiles/roofline_consts.json gets, per kernel, the
thread-instruction count and DRAM traffic per present pair (sample_kernel)
or per occurrence (compact_kernel): bench.py multiplies them by the units of
a launch and divides by the live CUDA-event kernel time.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import re
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
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_st.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def read_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [{h: (r[i], units[i]) for i, h in enumerate(hdr)} for r in rows[2:]]


def to_float(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def summarise(kern, units_per_launch):
    sel = {k: {"value": kern[k][0], "unit": kern[k][1]} for k in KEYS if k in kern}
    stalls = {h: v for h, (v, u) in kern.items() if "average_warps_issue_stalled" in h and h.endswith("ratio")
              and (to_float(v) or 0) > 0.1}
    inst = to_float(sel["smsp__inst_executed.sum"]["value"])
    if "smsp__thread_inst_executed.sum" in sel:
        t_inst = to_float(sel["smsp__thread_inst_executed.sum"]["value"])
    else:   # the full set carries the per-instruction thread ratio instead
        t_inst = inst * to_float(sel["smsp__thread_inst_executed_per_inst_executed.ratio"]["value"])
    scale = {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9, "s": 1.0}
    dur = to_float(sel["gpu__time_duration.sum"]["value"]) * scale[sel["gpu__time_duration.sum"]["unit"]]

    def bytes_of(k):
        v, u = to_float(sel[k]["value"]), sel[k]["unit"]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    dram = bytes_of("dram__bytes_read.sum") + bytes_of("dram__bytes_write.sum")
    derived = {"kernel": kern.get("Kernel Name", ("?", ""))[0], "duration_s": dur,
               "units_per_launch": units_per_launch, "thread_inst": t_inst, "warp_inst": inst,
               "thread_inst_per_unit": t_inst / units_per_launch,
               "dram_bytes": dram, "dram_bytes_per_unit": dram / units_per_launch,
               "lane_inst_per_s": t_inst / dur}
    return {"metrics": sel, "stalls": stalls, "derived": derived}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--pairs", type=float, required=True, help="present pairs in the profiled launch")
    ap.add_argument("--occurrences", type=float, required=True, help="YET occurrences in the profiled launch")
    ap.add_argument("--write-const", action="store_true")
    a = ap.parse_args()
    consts_path = os.path.join(ROOT, "profiles", "roofline_consts.json")
    consts = json.load(open(consts_path)) if os.path.exists(consts_path) else {}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    for kern in read_raw(a.rep):
        name = kern.get("Kernel Name", ("?", ""))[0]
        m = re.search(r"(compact_kernel|sample_kernel|scan_kernel|primary_kernel)", name)
        if not m:
            continue
        short = m.group(1)
        units = a.occurrences if short in ("compact_kernel", "primary_kernel") else a.pairs
        out = summarise(kern, units)
        out["source"] = os.path.basename(a.rep)
        with open(os.path.join(ROOT, "profiles", f"{a.tag}_{short}.json"), "w") as f:
            json.dump(out, f, indent=1)
        d = out["derived"]
        print(json.dumps({short: d}, indent=1))
        if a.write_const:
            key = "occurrence" if short in ("compact_kernel", "primary_kernel") else "pair"
            mm = out["metrics"]
            pick = lambda k: float(mm[k]["value"]) if k in mm else None
            consts[short] = {f"thread_inst_per_{key}": d["thread_inst_per_unit"],
                             f"dram_bytes_per_{key}": d["dram_bytes_per_unit"],
                             # L2 hit rate, pipe utilisation, issue, SM clock of the capture
                             "ncu": {"l2_hit_rate_pct": pick("lts__t_sector_hit_rate.pct"),
                                     "issue_active_pct": pick("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                                     "fma_pipe_pct": pick("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
                                     "alu_pipe_pct": pick("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                                     "xu_pipe_pct": pick("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
                                     "l1_lsu_wavefronts_pct": pick("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
                                     "l2_throughput_pct": pick("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                                     "dram_throughput_pct": pick("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
                                     "sm_ghz": pick("sm__cycles_elapsed.avg.per_second")},
                             "source": f"profiles/{a.tag}_{short}.json ({os.path.basename(a.rep)})"}
    if a.write_const:
        consts["source"] = f"profiles/{a.tag}_*.json"
        consts["note"] = "ncu --set full --clock-control none, one launch of each kernel on the first 200k trials of cfg3 (tools/capture_profiles.sh)"
        with open(consts_path, "w") as f:
            json.dump(consts, f, indent=1)


if __name__ == "__main__":
    main()
