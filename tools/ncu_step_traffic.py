"""Per-kernel DRAM traffic, L2 sectors and instruction counts of one hot-path step from an
`ncu --set full` capture of tools/perf_step.py -> profiles/ncu_traffic_<round>.json (read by bench.py
for roofline.traffic and roofline.stages).  Launches are tagged like libgod's profiler: the first
K1 launch is extract_ref, the second extract_phase; k_anchor_count is k_probe.
usage: python tools/ncu_step_traffic.py REPORT OUT_JSON"""
import csv
import json
import os
import re
import subprocess
import sys

rep, dst = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "sector": 1, "Ksector": 1e3,
         "Msector": 1e6, "Gsector": 1e9, "inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9, "nsecond": 1e-6,
         "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "%": 1}


def val(r, name):
    if name not in hdr:
        return None
    i = hdr.index(name)
    try:
        return float(r[i].replace(",", "")) * scale.get(units[i], 1.0)
    except ValueError:
        return None


ALIAS = {"k_anchor_count": "k_probe", "k_anchor_write1": "k_anchor_write", "k_rs_scatter2": "k_rs_scatter"}
seen = {}
res = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    m = re.search(r"(k_[A-Za-z0-9_]+|scan_[A-Za-z0-9_]+)", name)
    base = m.group(1) if m else name[:40]
    if base == "k_extract3" or base == "k_extract":
        i = seen.get("extract", 0)
        seen["extract"] = i + 1
        tag = ["extract_ref", "extract_phase"][i] if i < 2 else "extract_seed"
    else:
        tag = ALIAS.get(base, base)
    rd, wr = val(r, "dram__bytes_read.sum") or 0.0, val(r, "dram__bytes_write.sum") or 0.0
    e = res.setdefault(tag, {"launches": 0, "dram_read": 0.0, "dram_write": 0.0, "ncu_ms": 0.0, "l2_read_sectors": 0.0,
                             "inst_executed": 0.0, "kernel": name[:100]})
    e["launches"] += 1
    e["dram_read"] += rd
    e["dram_write"] += wr
    e["ncu_ms"] += val(r, "gpu__time_duration.sum") or 0.0
    e["l2_read_sectors"] += val(r, "lts__t_sectors_srcunit_tex_op_read.sum") or 0.0
    e["inst_executed"] += val(r, "smsp__inst_executed.sum") or 0.0
    hr = val(r, "lts__t_sector_hit_rate.pct")
    if hr is not None:
        e["l2_hit_rate_pct"] = round(hr, 2)
for tag, e in res.items():
    n = e["launches"]
    e["dram_bytes_per_launch"] = int((e["dram_read"] + e["dram_write"]) / n)
    for f in ("dram_read", "dram_write", "l2_read_sectors", "inst_executed"):
        e[f] = int(e[f] / n)
    e["ncu_ms_per_launch"] = round(e.pop("ncu_ms") / n, 4)
    e["source"] = os.path.basename(rep) + " (ncu --set full --clock-control none, one step of tools/perf_step.py)"
json.dump(res, open(dst, "w"), indent=1)
for tag, e in sorted(res.items(), key=lambda kv: -kv[1]["ncu_ms_per_launch"] * kv[1]["launches"]):
    print(f"{tag:22s} x{e['launches']} {e['ncu_ms_per_launch']:8.3f} ms  dram {e['dram_bytes_per_launch']/1e9:7.3f} GB  "
          f"l2rd {e['l2_read_sectors']/1e6:9.1f} Msec  inst {e['inst_executed']/1e9:6.3f} G")
