"""Fill BASELINE.md §3: run bench.py for every config / pattern (GPU, device-resident, 1 B200) with the
oracle baseline leg, and print one markdown row per workload.  Usage (on the GPU box):
    python tools/measure_table.py > gpurun_out/table.md"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROWS = [("Tiny '10'", "tiny"), ("Illumina '10'", "illumina"), ("HiFi '10'", "hifi"), ("HiFi '110'", "hifi-110"),
        ("ONT '10'", "ont"), ("Human '10'", "human"), ("Human '110'", "human-110"), ("Human '1110'", "human-1110"),
        ("Human '1'", "human-1")]
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
print("| Config / pattern | Index build Gbp/s | Stage 1+2 GB/s (% of 6.53 TB/s; of 8 TB/s) | Stage 3 ms (sort, count, "
      "cutoff, table) | Reads/s | Anchors/s | Step ms | Voting ms (reads/s) | Oracle (1 core) reads/s (sample) | Bit-exact |")
print("|---|---|---|---|---|---|---|---|---|---|")
for label, wl in ROWS:
    steps = "3" if wl.startswith("human") else "5"
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", wl, "--steps", steps, "--warmup", "3",
           "--no-e2e"]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
    try:
        d = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception:
        print(f"| {label} | failed: {out.stderr[-200:]!r} |")
        continue
    ks = d["kernels"]
    ex = ks.get("extract_ref", {}).get("ms_per_step", float("nan"))
    ref_bp = d["config"]["ref_bp"]
    byt = ref_bp + 12 * d["index"]["n_entries_all"]
    gbs = byt / (ex / 1e3) / 1e9
    st3 = d["stage_ms"]["index_build"] - ex
    cpu = d.get("cpu_baseline") or {}
    exact = "yes (full parity: tests/test_gpu_fullsize.py, test_gpu_parity.py)" if not wl.startswith("human") else \
        "yes on sampled outputs + properties (tests/test_gpu_fullsize.py)"
    print(f"| {label} | {d['index_build_gbps']:.1f} | {gbs:.0f} ({100 * gbs / PEAK:.1f}%; {100 * gbs / 8000:.1f}%) | "
          f"{st3:.1f} | {d['seed_reads_per_s'] / 1e6:.1f} M | {d['anchors_per_s'] / 1e9:.2f} G | {d['ms_per_step']:.2f} | "
          f"{(d.get('vote') or {}).get('ms', float('nan')):.2f} ({(d.get('vote') or {}).get('reads_per_s', float('nan')) / 1e6:.1f} M) | "
          f"{cpu.get('value', float('nan')):.0f} | {exact} |", flush=True)
