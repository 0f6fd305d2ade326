"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel: total time and
share of the profiled launches, next to the shares bench.py measured live (CUDA events).
usage: python tools/launch_share.py LAUNCHES.csv [BENCH.json]"""
import csv, json, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
iK, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot = defaultdict(float); cnt = defaultdict(int)
for r in rows[1:]:
    name = r[iK].split("(")[0].replace("void ", "").replace("unnamed>::", "").replace("god::", "")
    tot[name] += float(r[iV]) / 1e6
    cnt[name] += 1
T = sum(tot.values())
bench = {}
if len(sys.argv) > 2:
    b = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    ks = b["kernels"]; BT = sum(v["ms_per_step"] for v in ks.values())
    bench = {k: v["ms_per_step"] / BT for k, v in ks.items()}
print(f"{'kernel (ncu launch list)':40s} {'launches':>8s} {'ms':>9s} {'share':>7s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:40s} {cnt[k]:8d} {tot[k]:9.3f} {tot[k] / T * 100:6.2f}%")
print(f"{'total':40s} {sum(cnt.values()):8d} {T:9.3f}")
if bench:
    print("\nbench.py live shares (CUDA events, tag names):")
    for k, v in sorted(bench.items(), key=lambda kv: -kv[1])[:12]:
        print(f"  {k:30s} {v * 100:6.2f}%")
