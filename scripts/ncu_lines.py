"""Top source lines by warp-stall samples from an ncu report (development tool).
usage: python scripts/ncu_lines.py report.ncu-rep [n]"""
import csv
import subprocess
import sys

rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True,
                     text=True).stdout
cur, hdr, data = None, None, []
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0] not in ("",):  # source-line rows (SASS rows have an empty line no)
        d = {"line": r[0], "src": r[1], "file": cur}
        for i, c in enumerate(hdr[4:], 4):
            d.setdefault(c, r[i])
        data.append(d)


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


key = "Warp Stall Sampling (All Samples)"
tot = sum(f(d.get(key, 0)) for d in data) or 1.0
stall_cols = [c for c in (hdr or []) if c.startswith("stall_") and "Not Issued" not in c]
for d in sorted(data, key=lambda d: -f(d.get(key, 0)))[:n]:
    top = sorted(((f(d[c]), c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{f(d[key]) / tot * 100:5.1f}% {d['file'].split('/')[-1]}:{d['line']} "
          f"[{' '.join(f'{c}={v:.0f}' for v, c in top)}] {d['src'].strip()[:80]}")
