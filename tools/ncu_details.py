"""Selected per-launch metrics from an ncu report's details page.
usage: python tools/ncu_details.py REPORT [metric-name-substring ...]"""
import csv
import subprocess
import sys
from collections import OrderedDict

rep = sys.argv[1]
want = sys.argv[2:] or ["Duration", "DRAM Throughput", "Memory Throughput", "Issue Slots Busy", "Registers Per Thread",
                        "Achieved Occupancy", "Executed Ipc Active", "L2 Hit Rate"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
iid, ik, isec, iname, iu, iv = (hdr.index(c) for c in ("ID", "Kernel Name", "Section Name", "Metric Name", "Metric Unit",
                                                       "Metric Value"))
per = OrderedDict()
for r in rows[1:]:
    if len(r) <= iv:
        continue
    key = (r[iid], r[ik].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[:40])
    if any(w == r[iname] for w in want):
        per.setdefault(key, OrderedDict())[r[iname]] = f"{r[iv]} {r[iu]}".strip()
for (i, k), m in per.items():
    print(i, k, "|", "; ".join(f"{a}={b}" for a, b in m.items()))
