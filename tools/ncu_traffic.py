"""Per-launch DRAM traffic of profiled kernels from an `ncu --set full` report -> profiles/ncu_traffic_r01.json
(read by bench.py for roofline.traffic).
usage: python tools/ncu_traffic.py REPORT TAG:ROW [TAG:ROW ...]   (ROW = launch index in the report)"""
import csv, json, os, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
data = rows[2:]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
def val(r, name):
    i = hdr.index(name)
    return float(r[i]) * scale.get(units[i], 1.0)
dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic_r01.json")
res = json.load(open(dst)) if os.path.exists(dst) else {}
for spec in sys.argv[2:]:
    tag, row = spec.split(":")
    r = data[int(row)]
    rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
    res[tag] = {"dram_bytes_per_launch": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
                "kernel": r[hdr.index("Kernel Name")][:120], "source": os.path.basename(rep)}
    print(tag, res[tag])
json.dump(res, open(dst, "w"), indent=1)
