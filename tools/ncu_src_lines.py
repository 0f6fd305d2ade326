"""Per-source-line warp instructions / stall samples of one kernel from an ncu report (the CUDA-line
aggregate rows of the mixed cuda,sass source page; SASS rows are not double counted), plus optional
section totals over line ranges of one file.
usage: python tools/ncu_src_lines.py REPORT KERNEL_REGEX [N] [units] [file:lo-hi=name ...]
  units: divide instruction counts by this (e.g. positions) to print per-unit thread slots (x32)."""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
units = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
secs = []
for s in sys.argv[5:]:
    f, rest = s.split(":", 1)
    rng, name = rest.split("=", 1)
    lo, hi = map(int, rng.split("-"))
    secs.append((f, lo, hi, name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                      "regex:" + kre, "--launch-count", "1"], capture_output=True, text=True).stdout
fpath, hdr = "?", None
ins, samp, src = defaultdict(float), defaultdict(float), {}
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fpath = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        iS, iX = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        continue
    if hdr is None or not r[0] or len(r) <= iX:
        continue

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    key = (fpath, int(r[0]))
    ins[key] += f(r[iX])
    samp[key] += f(r[iS])
    src[key] = r[1]
TI, TS = sum(ins.values()) or 1, sum(samp.values()) or 1
per = (lambda x: f"  {32 * x / units:7.2f}/unit") if units else (lambda x: "")
print(f"total warp instructions {TI:.0f}{per(TI)}  samples {TS:.0f}")
for k in sorted(ins, key=lambda k: -ins[k])[:N]:
    print(f"{k[0][:12]:12s}:{k[1]:5d} {ins[k] / TI * 100:5.1f}% inst={ins[k]:12.0f}{per(ins[k])} samp={samp[k] / TS * 100:5.1f}%  "
          f"{src[k].strip()[:70]}")
if secs:
    print("sections:")
    acc = defaultdict(float)
    for k, v in ins.items():
        name = next((n for f, lo, hi, n in secs if k[0] == f and lo <= k[1] <= hi), "other:" + k[0])
        acc[name] += v
    for n in sorted(acc, key=lambda n: -acc[n]):
        print(f"  {n:28s} {acc[n] / TI * 100:5.1f}%{per(acc[n])}")
