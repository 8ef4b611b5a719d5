"""Per-kernel table from an ncu --csv --metrics launch list (development tool).
usage: python scripts/launch_table.py launches.csv"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit")}
k = OrderedDict()
for r in rows[1:]:
    key = (r[ix["ID"]], r[ix["Kernel Name"]].split("(")[0][:48])
    k.setdefault(key, {})[r[ix["Metric Name"]]] = (r[ix["Metric Value"]].replace(",", ""), r[ix["Metric Unit"]])
for (i, name), m in k.items():
    print(i, name, "  ".join(f"{a.split('__')[1].split('.')[0]}={v}{u}" for a, (v, u) in m.items()))
