#!/usr/bin/env python3
"""Extracts the judged numbers from ncu reports into profiles/ncu_summary.json.

usage: python profiles/summarize_ncu.py <stage>=<report.ncu-rep> [...] [--launches launches.csv]
  stage: "score" / "progressive" (the names bench.py uses for roofline.kernel)

Per kernel: duration, DRAM bytes read/written per launch (the roofline `traffic`),
DRAM / SM throughput, occupancy, registers, top stall reasons and pipe utilisation.
"""
import csv
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def ncu_page(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def summarize(rep):
    rows = ncu_page(rep, "raw")
    h, v = rows[0], rows[2]
    raw = dict(zip(h, v))
    det = {}
    for r in ncu_page(rep, "details"):
        if len(r) >= 3:
            det[r[-3]] = r[-1]
    g = lambda k: num(raw.get(k))  # noqa: E731
    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): g(k)
              for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")}
    stalls = {k: v for k, v in sorted(stalls.items(), key=lambda kv: -(kv[1] or 0)) if (v or 0) > 0.1}
    rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    unit_scale = 1.0
    # ncu reports bytes in the unit of the column header; raw page uses plain bytes for .sum counters
    return dict(
        kernel=raw.get("Kernel Name", "")[:120],
        duration_ms=(g("gpu__time_duration.sum") or 0) / 1e6,
        dram_bytes_read=rd * unit_scale if rd is not None else None,
        dram_bytes_write=wr * unit_scale if wr is not None else None,
        dram_bytes_per_launch=(rd or 0) + (wr or 0),
        dram_throughput_pct=num(det.get("DRAM Throughput")),
        sm_throughput_pct=num(det.get("Compute (SM) Throughput")),
        ipc=num(det.get("Executed Ipc Active")),
        achieved_occupancy_pct=num(det.get("Achieved Occupancy")),
        registers=num(det.get("Registers Per Thread")),
        pipes_pct={k.split(".")[0].replace("sm__", ""): g(k) for k in [
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"] if g(k) is not None},
        stalls_per_issue=stalls,
        report=os.path.basename(rep),
    )


def main():
    out_path = os.path.join(HERE, "ncu_summary.json")
    summary = json.load(open(out_path)) if os.path.exists(out_path) else {"kernels": {}}
    args = sys.argv[1:]
    for a in args:
        if "=" in a:
            stage, rep = a.split("=", 1)
            summary["kernels"][stage] = summarize(rep)
    summary["note"] = ("dram bytes are per launch from `ncu --set full --clock-control none` (cold cache, "
                       "serialised replay): compare shares and traffic, not absolute times")
    json.dump(summary, open(out_path, "w"), indent=1)
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main()
