"""Per-source-line stall samples / instructions from an ncu report (cuda,sass mixed source page).
usage: python tools/ncu_lines.py REPORT [N] [KERNEL_REGEX] [LAUNCH_SKIP]"""
import csv, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
flt = ["--kernel-name", "regex:" + sys.argv[3], "--launch-count", "1"] if len(sys.argv) > 3 else []
if len(sys.argv) > 4:
    flt += ["--launch-skip", sys.argv[4]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + flt,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iX = hdr.index("Instructions Executed")
samp, ins, src = defaultdict(float), defaultdict(float), {}
line = None
for r in rows[hi + 1:]:
    if len(r) <= iS:
        continue
    if r[0] == "Line No":
        continue
    if r[0]:
        line = int(r[0]); src[line] = r[1]
    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    samp[line] += f(r[iS]); ins[line] += f(r[iX])
tot = sum(samp.values()) or 1
print(f"total samples {tot:.0f}  instructions {sum(ins.values()):.0f}")
for l in sorted(samp, key=lambda l: -samp[l])[:N]:
    print(f"{l:5d} {samp[l] / tot * 100:5.1f}%  inst={ins[l]:12.0f}  {src.get(l, '').strip()[:90]}")
