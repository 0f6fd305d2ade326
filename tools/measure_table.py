"""Fill BASELINE.md §3: run bench.py for every config / pattern (GPU, device-resident, 1 B200) and
print two markdown tables:
  (1) GPU throughput per workload, with the bit-exact column taken from the whole-config digest
      parity log (tests/test_gpu_digests.py -> parity_digests.jsonl), not asserted here;
  (2) the CPU oracle stage by stage over the WHOLE workload (tests/golden/digests/<row>.json, written by
      tools/oracle_digests.py: time.perf_counter per stage, 1 core, host model and nproc recorded)
      against the GPU stage times, with the GPU/oracle speedup per stage.
Usage (on the GPU box, after `pytest tests/test_gpu_digests.py -m gpu`):
    python tools/measure_table.py [parity_digests.jsonl] > gpurun_out/table.md"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROWS = [("Tiny '10'", "tiny", "tiny_10"), ("Illumina '10'", "illumina", "illumina_10"), ("HiFi '10'", "hifi", "hifi_10"),
        ("HiFi '110'", "hifi-110", "hifi_110"), ("ONT '10'", "ont", "ont_10"), ("Human '10'", "human", "human_10"),
        ("Human '110'", "human-110", "human_110"), ("Human '1110'", "human-1110", "human_1110"),
        ("Human '1'", "human-1", "human_1")]
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
log = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "parity_digests.jsonl")
parity = {}
if os.path.exists(log):
    for line in open(log):
        try:
            d = json.loads(line)
        except ValueError:
            continue
        if "call" in d:  # the host-call digest rows (test_digest_parity_host_call) are not table rows
            continue
        parity[f"{d['config']}_{d['pattern']}"] = d  # the last run of a row wins


def exact(key):
    d = parity.get(key)
    if d is None:
        return "not run"
    if d["bit_exact"]:
        return f"yes ({len(d['compared'])}/{len(d['compared'])} digests, test_gpu_digests.py)"
    return "NO: " + "; ".join(d["failures"])[:120]


def gold(key):
    p = os.path.join(ROOT, "tests", "golden", "digests", key + ".json")
    return json.load(open(p)) if os.path.exists(p) else None


bench = {}
for label, wl, key in ROWS:
    steps = "3" if wl.startswith("human") else "5"
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", wl, "--steps", steps, "--warmup", "3",
           "--no-e2e", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
    try:
        bench[key] = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception:
        bench[key] = {"error": out.stderr[-200:]}

print(f"| Config / pattern | Index build Gbp/s | Stage 1+2 GB/s (% of {PEAK / 1e3:.2f} TB/s; of 8 TB/s) | Stage 3 ms "
      "(% of floor rate) | Reads/s | Anchors/s | Step ms | Voting ms (reads/s) | Bit-exact (whole config) |")
print("|---|---|---|---|---|---|---|---|---|")
for label, wl, key in ROWS:
    d = bench[key]
    if "error" in d:
        print(f"| {label} | failed: {d['error']!r} |")
        continue
    st = (d.get("roofline") or {}).get("stages", {})
    s12, s3 = st.get("stage12_sparsify_extract", {}), st.get("stage3_index", {})
    v = d.get("vote") or {}
    print(f"| {label} | {d['index_build_gbps']:.1f} | {s12.get('achieved_gbs', float('nan')):.0f} "
          f"({100 * s12.get('frac', float('nan')):.1f}%; {100 * s12.get('frac_of_8tbs', float('nan')):.1f}%) | "
          f"{s3.get('ms', float('nan')):.1f} ({100 * s3.get('frac', float('nan')):.1f}%) | "
          f"{d['seed_reads_per_s'] / 1e6:.1f} M | {d['anchors_per_s'] / 1e9:.2f} G | {d['ms_per_step']:.2f} | "
          f"{v.get('ms', float('nan')):.2f} ({v.get('reads_per_s', float('nan')) / 1e6:.1f} M) | {exact(key)} |", flush=True)

print()
print("| Config / pattern | Oracle: sparsify ref s | minimizers ref s | index build s | phase selection s | "
      "seeding s | GPU: stage 1+2 ms | index build ms | phase sel. + seeding ms | Speedup: index build | "
      "phase sel. + seeding | Oracle host |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for label, wl, key in ROWS:
    g, d = gold(key), bench.get(key, {})
    if g is None or "error" in d:
        print(f"| {label} | (no oracle digest run) |")
        continue
    t = g["timing_s"]
    ks = d["kernels"]
    s12 = ks.get("extract_ref", {}).get("ms_per_step", float("nan"))
    bms, sms = d["stage_ms"]["index_build"], d["stage_ms"]["phase_select_and_seed"]
    ps = t.get("phase_select", float("nan"))
    sg = t.get("seed_given", float("nan"))
    h = g.get("host", {})
    print(f"| {label} | {t['sparsify_ref']:.1f} | {t['extract_ref']:.1f} | {t['index_build']:.1f} | {ps:.1f} | {sg:.1f} | "
          f"{s12:.2f} | {bms:.2f} | {sms:.2f} | {t['index_build'] * 1e3 / bms:,.0f}x | "
          f"{t['select_and_seed'] * 1e3 / sms:,.0f}x | {h.get('cpu_model', '?')}, nproc {h.get('nproc', '?')}, 1 core |",
          flush=True)
