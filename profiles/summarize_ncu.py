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


UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6, "s": 1e3, "second": 1e3}


def summarize(rep):
    rows = ncu_page(rep, "raw")
    h, units, v = rows[0], rows[1], rows[2]
    raw = {k: (x, u) for k, u, x in zip(h, units, v)}

    def g(k, to_base=False):
        if k not in raw:
            return None
        x, u = raw[k]
        val = num(x)
        if val is None:
            return None
        return val * UNIT.get(u, 1.0) if to_base else val

    det = {}
    for r in ncu_page(rep, "details")[1:]:
        if len(r) >= 15:
            det[r[12]] = (r[14], r[13])
    d = lambda k: num(det[k][0]) if k in det else None  # noqa: E731
    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): g(k)
              for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")}
    stalls = {k: v for k, v in sorted(stalls.items(), key=lambda kv: -(kv[1] or 0)) if (v or 0) > 0.1}
    rd, wr = g("dram__bytes_read.sum", True), g("dram__bytes_write.sum", True)
    return dict(
        kernel=raw.get("Kernel Name", ("",))[0][:120],
        duration_ms=g("gpu__time_duration.sum", True),
        dram_bytes_read=rd,
        dram_bytes_write=wr,
        dram_bytes_per_launch=(rd or 0) + (wr or 0),
        dram_throughput_pct_of_nominal=d("DRAM Throughput"),
        sm_throughput_pct=d("Compute (SM) Throughput"),
        ipc=d("Executed Ipc Active"),
        achieved_occupancy_pct=d("Achieved Occupancy"),
        registers=d("Registers Per Thread"),
        sm_clock_ghz=d("SM Frequency"),
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
