"""Per-role totals (instructions executed, stall samples) of the warp-specialised stream kernel from an
ncu report with source (development tool). usage: python scripts/role_split.py report.ncu-rep P,D,S,V (banner line numbers)"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr = None, None
rows = []
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0] not in ("", "-") and cur and cur.endswith("kernels_stream.cu"):
        d = {"Line No": r[0], "Source": r[1]}
        for i, c in enumerate(hdr[4:], 4):
            d.setdefault(c, r[i])
        rows.append((int(r[0]), r[1], d))
markers = [("producer", "PRODUCER"), ("decider", "DECIDER"), ("scorer", "SCORERS"), ("v", "== V ==")]
# role boundaries: source lines of the role banners (comment lines carry no SASS), given as
# producer,decider,scorer,v line numbers of the captured source
bounds = list(zip(map(int, sys.argv[2].split(",")), [m[0] for m in markers]))


def role(ln):
    r = "setup"
    for b, name in bounds:
        if ln >= b:
            r = name
    return r


def num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


tot = {}
for ln, src, d in rows:
    rl = role(ln)
    t = tot.setdefault(rl, [0.0, 0.0])
    t[0] += num(d.get("Instructions Executed", "0"))
    t[1] += num(d.get("Warp Stall Sampling (All Samples)", "0"))
I = sum(v[0] for v in tot.values()) or 1
S = sum(v[1] for v in tot.values()) or 1
print("role        instr(warp)   share   stall-samples share")
for k, (i, s) in tot.items():
    print(f"{k:10s} {i:14.0f} {100 * i / I:6.1f}% {s:12.0f} {100 * s / S:6.1f}%")
