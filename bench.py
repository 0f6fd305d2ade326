#!/usr/bin/env python
"""Benchmark of the Genome-on-Diet hot path on B200 (BASELINE.json metric).

A STEP is one pass of the whole hot path over one batch of synthetic input, all in libgod's CUDA
kernels through the C ABI: build the seed index of the reference (sparsify + minimizers + sort +
cutoff + table), then pattern alignment (phase selection) and compressed
seeding of every read.  Default workload = BASELINE configs[4] "human-scale" with the
paper's pattern '10': 3.1 Gbp repeat-rich synthetic reference + 10,000,000 x 150 bp reads,
k=21, w=11, cutoff top 0.02%.  Inputs (3.1 GB + 1.5 GB) are larger than L2 (126 MB), so no flush
is needed between steps.

value = reads seeded per second over the whole step (index build included), summed over ranks.
e2e   = the same through the C ABI from pinned HOST buffers, one god_build_index_and_seed call per
        step: the reference goes up in chunks while K1 runs on the tiles that are in, the read
        batches follow on the same copy stream while the index is sorted, and each batch's 8-B
        anchors, offsets and phases stream back while later batches are seeded.  The last step's
        host results are compared with the device-resident step's (e2e.equals_device_step).
--impl reference: the CPU oracle (oracle/, plain single-threaded C) on a bounded sample of the
same workload, extrapolated to the metric's unit (see cpu_baseline.sample).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "seeded reads/s and index-build Gbp/s on 1 B200; % of HBM roofline"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")

WORKLOADS = {
    # name: (config, pattern, k, w)
    "human": ("human", "10", 21, 11),
    "human-110": ("human", "110", 21, 11),
    "human-1110": ("human", "1110", 21, 11),
    "human-1": ("human", "1", 21, 11),
    "illumina": ("illumina", "10", 21, 11),
    "hifi": ("hifi", "10", 19, 19),
    "hifi-110": ("hifi", "110", 19, 19),
    "ont": ("ont", "10", 15, 10),
    "tiny": ("tiny", "10", 21, 11),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="human", choices=sorted(WORKLOADS))
    ap.add_argument("--scale", type=float, default=1.0, help="size multiplier (1.0 = the BASELINE config)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-inputs", choices=["host", "host2", "staged"], default="host",
                    help="host: pinned host buffers into god_build_index_and_seed (default); host2: into the two "
                         "separate calls; staged: the caller copies the inputs to the device itself")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-vote", action="store_true")
    ap.add_argument("--vote-D", type=int, default=0, help="voting distance D (0 = read length)")
    ap.add_argument("--vote-V", type=int, default=3)
    ap.add_argument("--vote-max-pairs", type=int, default=0)
    ap.add_argument("--cpu-sample-bp", type=int, default=40_000_000)
    ap.add_argument("--cpu-sample-reads", type=int, default=40_000)
    return ap.parse_args()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------------------------------ data
def make_inputs(workload: str, scale: float, rank: int):
    import synth
    cfg_name, pattern, k, w = WORKLOADS[workload]
    t0 = time.time()
    cfg = synth.make_config(cfg_name, scale=scale, read_seed_offset=7919 * rank)
    log(f"[bench] rank {rank}: generated {cfg_name} x{scale}: ref {cfg.ref.size/1e9:.3f} Gbp, "
        f"{cfg.reads.n} reads ({cfg.reads.seq.size/1e9:.3f} Gbp) in {time.time()-t0:.1f}s")
    return cfg, pattern, k, w


# ------------------------------------------------------------------------------------------ multi-GPU plumbing
# Replicas: every rank builds the index of the same reference and seeds its OWN batch
# of reads (read seed offset by rank) -> weak scaling, no data-path collective.  The only collective
# is the max-over-ranks of the device-timed region.
def max_over_ranks(x: float, dist=None, device=None) -> float:
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_rate(units_per_rank: int, world: int, ms_per_step_max: float) -> float:
    """Whole-job throughput: the units all ranks processed / the slowest rank's time."""
    return world * units_per_rank / (ms_per_step_max / 1e3)


def workload_config(args, cfg, pattern, k, w, world):
    idx = {"tiny": 0, "illumina": 1, "hifi": 2, "hifi-110": 2, "ont": 3}.get(args.workload, 4)
    return {"workload": f"{args.workload}: BASELINE.json configs[{idx}] ({cfg.ref.size/1e9:.2f} Gbp reference, "
                        f"{cfg.reads.n} reads/rank, pattern '{pattern}', k={k}, w={w}, cutoff top "
                        f"{cfg.cutoff[0]}/{cfg.cutoff[1]})",
            "ref_bp": int(cfg.ref.size), "n_reads": cfg.reads.n, "read_bp": int(cfg.reads.seq.size),
            "pattern": pattern, "k": k, "w": w, "scale": args.scale,
            "l2_policy": "inputs larger than L2 (no flush needed)", "parallelism": f"replicas x{world} (weak)"}


# ------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        if os.environ.get("GOD_BENCH_NO_CLOCKS"):  # diagnostic: run without the sampler
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        med = float(np.median(sm)) if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------ roofline
EXTRACT_KERNELS = ("extract_ref", "extract_phase", "extract_seed")
# stage 1+2 (K1 on the reference) and the job set-up around it; everything else in the build is stage 3
STAGE12_BUILD = ("extract_ref", "k_make_jobs", "scan_jobs", "k_x2_tile_desc")
NOMINAL_HBM_GBS = 8000.0   # the north star's "~8 TB/s" (report against both)
G0_RANDOM_GATHER = {"64MB": 226.5e9, "512MB": 49.2e9, "4GB": 37.9e9}  # profiles/g0_microbench_r01.jsonl, sectors/s


def algorithmic_bytes(name: str, ctx: dict):
    """Algorithmic bytes per LAUNCH of the named kernel (DESIGN.md §5 table): what the method must
    move, not what a kernel happens to touch."""
    n_ref_mz = ctx["n_entries_all"]
    if name == "extract_ref":      # read every reference byte once; write 12 B per minimizer (u64 hash|strand, u32 pos)
        return ctx["ref_bytes"] + 12 * n_ref_mz
    if name in ("k_rs_scatter", "k_rs_scatter2"):  # read + write one 12-B record per pass
        return 24 * n_ref_mz
    if name == "k_rs_hist":
        return 8 * n_ref_mz
    if name == "extract_seed":     # read bytes once; write hz, pos, read id per read minimizer
        return ctx["read_bytes"] + 16 * ctx["n_read_mz"]
    if name == "extract_phase":
        return ctx["read_bytes"] + 12 * ctx["n_phase_mz"]
    return None


def load_traffic():
    """ncu-measured per-launch DRAM bytes, L2 sectors and instructions of one step (`ncu --set full`
    capture of tools/perf_step.py, summarised by tools/ncu_step_traffic.py); round 2 first."""
    for name in ("ncu_traffic_r02.json", "ncu_traffic_r01.json"):
        p = os.path.join(ROOT, "profiles", name)
        if os.path.exists(p):
            try:
                d = json.load(open(p))
                for v in d.values():
                    v.setdefault("file", "profiles/" + name)
                return d
            except Exception:
                pass
    return {}


def pick_roofline(prof: dict, ctx: dict, peaks: dict, units: dict, steps: int):
    """Headline roofline = the dominant kernel's HBM view (algorithmic bytes / measured launch time
    against the measured copy peak), plus roofline.stages: stage 1+2 (K1 on the reference), stage 3
    (index sort/cutoff/table: survey floor bytes / stage time, ncu bytes and passes) and stage 4
    (seeding: probes and 32-B sectors per second against G0's random-gather rates)."""
    items = sorted(prof.items(), key=lambda kv: -kv[1][0])
    total_ms = sum(v[0] for v in prof.values())
    peak_gbs = float(peaks.get("hbm_gbs", 6451.8))
    traffic = load_traffic()
    head = None
    for name, (ms, n) in items:
        b = algorithmic_bytes(name, ctx)
        if b is None:
            continue
        avg_s = ms / n / 1e3
        tr = traffic.get(name, {})
        ach = b / avg_s / 1e9
        head = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak_gbs, "unit": "GB/s", "frac": round(ach / peak_gbs, 4),
                "traffic": tr.get("dram_bytes_per_launch"), "kernel": name, "share_of_step": round(ms / total_ms, 4),
                "avg_launch_ms": round(avg_s * 1e3, 4), "algorithmic_bytes_per_launch": int(b),
                "frac_of_8tbs": round(ach / NOMINAL_HBM_GBS, 4),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, measured; burst)",
                "traffic_source": tr.get("file")}
        if name in EXTRACT_KERNELS and units.get(name):
            pos = units[name] / n
            head["positions_per_launch"] = int(pos)
            if tr.get("inst_executed"):  # measured instruction issue (the kernel is issue-bound)
                slots = 32.0 * tr["inst_executed"] / pos
                issue_floor_ms = tr["inst_executed"] / (148 * 4 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6) * 1e3
                head["issue_view"] = {"warp_inst_per_launch": tr["inst_executed"],
                                      "thread_slots_per_position": round(slots, 1),
                                      "issue_bound_ms_at_100pct": round(issue_floor_ms, 3),
                                      "frac_of_issue_peak": round(issue_floor_ms / (avg_s * 1e3), 4),
                                      "source": tr.get("file")}
        break
    stages = {}
    ms_of = lambda t: prof.get(t, (0.0, 1))[0] / steps  # noqa: E731
    n = ctx["n_entries_all"]
    if "extract_ref" in prof:
        b = ctx["ref_bytes"] + 12 * n
        t = ms_of("extract_ref")
        stages["stage12_sparsify_extract"] = {
            "kernel": "extract_ref", "ms": round(t, 4), "algorithmic_bytes": int(b),
            "achieved_gbs": round(b / t / 1e6, 1), "frac": round(b / t / 1e6 / peak_gbs, 4),
            "frac_of_8tbs": round(b / t / 1e6 / NOMINAL_HBM_GBS, 4),
            "ncu_dram_bytes": traffic.get("extract_ref", {}).get("dram_bytes_per_launch")}
    s3 = {k: v for k, v in prof.items() if k in ctx["build_kernels"] and k not in STAGE12_BUILD}
    if s3:
        t = sum(v[0] for v in s3.values()) / steps
        floor = 12 * n + 8 * ctx["kept_entries"] + 16 * ctx["kept_distinct"] + 4 * (1 << ctx["dir_bits"])
        nb = sum(traffic[k]["dram_bytes_per_launch"] * (v[1] // steps) for k, v in s3.items() if k in traffic)
        stages["stage3_index"] = {
            "ms": round(t, 4), "floor_bytes": int(floor),
            "floor_def": "SURVEY §8(d): 12 B read per record + 8 B per kept entry + 16 B per kept distinct key + 4 B x 2^dir_bits",
            "achieved_gbs": round(floor / t / 1e6, 1), "frac": round(floor / t / 1e6 / peak_gbs, 4),
            "ncu_dram_bytes": int(nb) if nb else None,
            "ncu_bytes_over_floor": round(nb / floor, 2) if nb else None,
            "record_passes": round(nb / (24.0 * n), 2) if nb else None,
            "kernels_ms": {k: round(v[0] / steps, 4) for k, v in sorted(s3.items(), key=lambda kv: -kv[1][0])}}
    if "k_probe" in prof and units.get("k_probe"):
        t = ms_of("k_probe")
        probes = units["k_probe"] / steps
        tr = traffic.get("k_probe", {})
        sec = tr.get("l2_read_sectors")
        st4 = {"kernel": "k_probe", "ms": round(t, 4), "probes": int(probes), "probes_per_s": round(probes / t * 1e3, 1),
               "g0_random_gather_sectors_per_s": G0_RANDOM_GATHER}
        # each probe is one dependent random 32-B directory read (plus streaming record I/O): its
        # ceiling is G0's random 32-B gather rate over a buffer of the directory's size (4.2 GB here)
        st4["frac_of_g0_4gb_gather"] = round(probes / t * 1e3 / G0_RANDOM_GATHER["4GB"], 3)
        if sec:
            st4.update({"l2_read_sectors_per_probe": round(sec / probes, 2),
                        "dram_bytes_per_probe": round(tr["dram_bytes_per_launch"] / probes, 1),
                        "algorithmic_bytes_per_probe": 32 + 8 + 8,  # directory sector + record in + (count, first) out
                        "l2_hit_rate_pct": tr.get("l2_hit_rate_pct"), "source": tr.get("file")})
        if "k_anchor_write" in prof:
            ta = ms_of("k_anchor_write")
            st4["anchor_write"] = {"ms": round(ta, 4), "anchors_per_s": round(ctx["n_anchors"] / ta * 1e3, 1),
                                   "ncu_dram_bytes": traffic.get("k_anchor_write", {}).get("dram_bytes_per_launch"),
                                   "algorithmic_bytes": 16 * ctx["n_anchors"]}
        stages["stage4_seeding"] = st4
    if head is not None:
        head["stages"] = stages
    return head


# ------------------------------------------------------------------------------------------ CPU oracle
def host_info() -> dict:
    model = ""
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def oracle_sample(cfg, pattern, k, w, sample_bp: int, sample_reads: int):
    """Time the CPU oracle (single thread, as it stands) stage by stage on a bounded sample: a
    reference prefix of sample_bp bases (stage 1 sparsify, stage 2 minimizers, stage 1-3 index) and
    sample_reads reads simulated from it (stage 4: SELECT-mode phase selection + seeding, and
    GIVEN-mode seeding alone, so phase selection = the difference).  Each stage is extrapolated
    linearly to the full workload (reference bases, reads).  Returns (seconds for the whole step
    extrapolated, description, seconds spent, per-stage dict)."""
    import oracle
    import synth
    L = min(sample_bp, cfg.ref.size)
    pref = np.ascontiguousarray(cfg.ref[:L])
    off = np.array([0, L], np.uint64)
    fr = cfg.ref.size / L
    t0 = time.perf_counter()
    oracle.sparsify(pref, pattern, 0)
    t_sp = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.minimizers_batch(pref, off, pattern, k, w, global_pos=True)
    t_mz = time.perf_counter() - t0
    t0 = time.perf_counter()
    ix = oracle.Index(pref, off, pattern, k, w)
    t_idx = time.perf_counter() - t0
    rd = cfg.reads
    nr = min(sample_reads, rd.n)
    fq = rd.n / max(1, nr)
    lens = np.diff(rd.offsets.astype(np.int64))
    mean_len = float(lens.mean()) if lens.size else 150.0
    sim = synth.simulate_reads(pref, nr, 9001, length=int(round(mean_len)), start_margin=int(mean_len * 1.3) + 64,
                               p_sub=0.001, p_ins=0.00005, p_del=0.00005)
    t0 = time.perf_counter()
    _, _, ph = ix.seed_reads(sim.seq, sim.offsets)
    t_seed = time.perf_counter() - t0
    t0 = time.perf_counter()
    ix.seed_reads(sim.seq, sim.offsets, phases=ph)
    t_given = time.perf_counter() - t0
    full = t_idx * fr + t_seed * fq
    stages = {  # seconds for the full workload, extrapolated linearly from the sample
        "stage1_sparsify_ref_s": round(t_sp * fr, 2),
        "stage2_minimizers_ref_s": round(t_mz * fr, 2),
        "stage3_index_build_s": round(t_idx * fr, 2),   # includes its own stage 1+2 pass (oracle.c or_build_index)
        "stage4a_phase_select_s": round(max(0.0, t_seed - t_given) * fq, 2),
        "stage4b_seeding_s": round(t_given * fq, 2),
        "extrapolated": True, "sample_ref_bp": int(L), "sample_reads": int(nr), **host_info(), "cores_used": 1}
    desc = (f"oracle stage by stage on a {L/1e6:.0f} Mbp reference prefix (sparsify {t_sp:.1f}s, minimizers {t_mz:.1f}s, "
            f"index {t_idx:.1f}s) and {nr} reads simulated from it (SELECT seeding {t_seed:.1f}s, GIVEN seeding "
            f"{t_given:.1f}s), each extrapolated linearly to the full workload ({cfg.ref.size/1e9:.2f} Gbp, {rd.n} reads)")
    return full, desc, t_sp + t_mz + t_idx + t_seed + t_given, stages


# ------------------------------------------------------------------------------------------ main
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, world, rank)
    import torch
    import paper_2211_08157_b200 as god
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    cfg, pattern, k, w = make_inputs(args.workload, args.scale, rank)
    n_reads = cfg.reads.n
    dref = torch.from_numpy(cfg.ref).to(dev)
    droff = torch.from_numpy(cfg.ref_offsets).to(dev)
    dreads = torch.from_numpy(cfg.reads.seq).to(dev)
    droffs = torch.from_numpy(cfg.reads.offsets).to(dev)
    torch.cuda.synchronize()

    outbuf = {}

    def step(cap=None, ev=None):
        if ev:
            ev[0].record()
        ix = god.god_build_index(dref, droff, pattern, k, w, cutoff=cfg.cutoff)
        if ev:
            ev[1].record()
        if cap is not None and "an" not in outbuf:  # steady state: preallocated outputs, no allocation per step
            outbuf["an"] = torch.empty((cap, 4), dtype=torch.uint32, device=dev)
            outbuf["ao"] = torch.empty(n_reads + 1, dtype=torch.uint64, device=dev)
            outbuf["ph"] = torch.empty(max(1, n_reads), dtype=torch.uint8, device=dev)
        out = (outbuf["an"], outbuf["ao"], outbuf["ph"]) if cap is not None else None
        an, ao, ph = god.god_seed_reads(ix, dreads, droffs, cap=cap, out=out)
        if ev:
            ev[2].record()
        st = ix.stats()
        ix.free()  # a step builds, uses and releases its index (the pool keeps the memory mapped)
        return st, an

    # warm-up (also sizes the anchor output)
    cap = None
    for i in range(max(args.warmup, 1)):
        st, an = step(cap)
        cap = max(int(an.shape[0]), 1)
        del an
    n_anchors = cap
    torch.cuda.synchronize()

    # timed region
    god.profile_reset()
    god.profile_enable(True)
    launches0 = god.launch_count()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(torch.cuda.current_device())
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk.start()
    start.record()
    for i in range(args.steps):
        st, an = step(cap, evs[i])
    end.record()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = clk.stop()
    god.profile_enable(False)
    launches = god.launch_count() - launches0
    prof = god.profile_query()
    units = {kname: god.profile_units(kname) for kname in EXTRACT_KERNELS + ("k_probe",)}
    elapsed_ms = start.elapsed_time(end)
    build_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in evs]))
    seed_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in evs]))
    log("[bench] per-step build/seed ms: " + " ".join(f"{e[0].elapsed_time(e[1]):.1f}/{e[1].elapsed_time(e[2]):.1f}"
                                                      for e in evs))
    elapsed_ms = max_over_ranks(elapsed_ms, dist, dev)
    ms_per_step = elapsed_ms / args.steps
    value = aggregate_rate(n_reads, world, ms_per_step)

    # which kernels belong to the index build (stage 1+2 + stage 3), from one untimed profiled build
    god.profile_reset()
    god.profile_enable(True)
    ixb = god.god_build_index(dref, droff, pattern, k, w, cutoff=cfg.cutoff)
    torch.cuda.synchronize()
    ixb.free()
    build_kernels = set(god.profile_query().keys())
    god.profile_enable(False)
    # records counts for the byte model (one extra untimed pass)
    hz, _, _, _ = god.god_minimizers(dreads, droffs, pattern, k, w, phases=None)  # phase-0 read minimizers (approx.)
    n_read_mz = int(hz.shape[0])
    del hz
    peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}
    ctx = {"ref_bytes": int(cfg.ref.size), "read_bytes": int(cfg.reads.seq.size), "n_entries_all": st["n_entries_all"],
           "n_read_mz": n_read_mz, "n_phase_mz": n_read_mz * 2, "kept_entries": st["kept_entries"],
           "kept_distinct": st["kept_distinct"], "dir_bits": st["dir_bits"], "n_anchors": n_anchors,
           "build_kernels": build_kernels}
    roof = pick_roofline(prof, ctx, peaks, units, args.steps)
    kernels = {kname: {"ms_per_step": round(ms / args.steps, 4), "launches_per_step": n // args.steps}
               for kname, (ms, n) in sorted(prof.items(), key=lambda kv: -kv[1][0])}

    # location voting: measured on the last step's anchors, separately
    # from the step (the §8(a) path ends at the anchors)
    vote = None
    if not args.no_vote:
        vote = run_vote(god, torch, dreads, droffs, dref, droff, cfg, pattern, k, w, args, dist, dev)

    # e2e through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(god, torch, cfg, pattern, k, w, n_anchors, args.e2e_steps, dist, world, dev, args.e2e_inputs,
                      outbuf)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        full_s, desc, spent, ostages = oracle_sample(cfg, pattern, k, w,
                                                     int(args.cpu_sample_bp * args.scale) or 1_000_000,
                                                     max(1000, int(args.cpu_sample_reads * args.scale)))
        gpu_s = {"stage12_extract_ref_s": prof.get("extract_ref", (0.0, 1))[0] / args.steps / 1e3,
                 "stage3_index_build_s": build_ms / 1e3, "stage4_phase_select_and_seed_s": seed_ms / 1e3}
        cpu = {"value": round(n_reads / full_s, 2), "unit": "reads/s", "cores": 1, "kind": "oracle",
               "sample": desc, "cpu_seconds_spent": round(spent, 1), "stages": ostages,
               "speedup_gpu_over_oracle": {
                   "stage1+2 (minimizers of the reference)": round(ostages["stage2_minimizers_ref_s"] / gpu_s["stage12_extract_ref_s"], 1)
                   if gpu_s["stage12_extract_ref_s"] else None,
                   "index build (stages 1-3)": round(ostages["stage3_index_build_s"] / gpu_s["stage3_index_build_s"], 1),
                   "phase selection + seeding (stage 4)": round((ostages["stage4a_phase_select_s"] + ostages["stage4b_seeding_s"])
                                                                / gpu_s["stage4_phase_select_and_seed_s"], 1)}}

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 1), "unit": "reads/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": workload_config(args, cfg, pattern, k, w, world),
            "index_build_gbps": round(cfg.ref.size / (build_ms / 1e3) / 1e9, 3),
            "seed_reads_per_s": round(n_reads / (seed_ms / 1e3), 1),
            "anchors_per_s": round(n_anchors / (seed_ms / 1e3), 1),
            "stage_ms": {"index_build": round(build_ms, 3), "phase_select_and_seed": round(seed_ms, 3)},
            "index": {kk: st[kk] for kk in ("n_entries_all", "n_distinct_all", "m", "tau", "kept_entries", "dir_bits")},
            "n_anchors_per_step": n_anchors,
            "roofline": roof, "kernels": kernels,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
            "vote": vote,
        }
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


def run_vote(god, torch, dreads, droffs, dref, droff, cfg, pattern, k, w, args, dist, dev):
    """Location voting (god_vote_reads) on the anchors of one seeding pass: W warm-up + K timed calls,
    CUDA events on the current stream, max over ranks.  HBM view: algorithmic bytes = every anchor
    read once (16 B) + every voted location written once (40 B) + read offsets/phases."""
    ix = god.god_build_index(dref, droff, pattern, k, w, cutoff=cfg.cutoff)
    an, ao, ph = god.god_seed_reads(ix, dreads, droffs)
    kw = dict(D=args.vote_D, V=args.vote_V, max_pairs=args.vote_max_pairs)
    for _ in range(max(args.warmup, 1)):
        v, vo = god.god_vote_reads(ix, dreads, droffs, ph, an, ao, **kw)
    torch.cuda.synchronize()
    god.profile_reset()
    god.profile_enable(True)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.steps):
        v, vo = god.god_vote_reads(ix, dreads, droffs, ph, an, ao, **kw)
    e.record()
    torch.cuda.synchronize()
    god.profile_enable(False)
    prof = god.profile_query()
    ms = max_over_ranks(s.elapsed_time(e) / args.steps, dist, dev)
    vv = god.votes_numpy(v)
    n = cfg.reads.n
    n_an = int(an.shape[0])
    kern = {kk: round(x[0] / args.steps, 4) for kk, x in sorted(prof.items(), key=lambda kv: -kv[1][0])}
    peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {"hbm_gbs": 6650.0}
    alg = 16 * n_an + 40 * int(vv.size) + 8 * 3 * (n + 1) + n
    ix.free()
    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    return {"params": kw, "ms": round(ms, 3), "reads_per_s": round(world * n / (ms / 1e3), 1),
            "anchors_per_s": round(world * n_an / (ms / 1e3), 1), "n_anchors": n_an, "n_locations": int(vv.size),
            "rescued": int(vv["rescued"].sum()), "kernels_ms": kern,
            "hbm_view": {"algorithmic_bytes": alg, "achieved_gbs": round(alg / (ms / 1e3) / 1e9, 1),
                         "peak_gbs": float(peaks.get("hbm_gbs", 6650.0)),
                         "frac": round(alg / (ms / 1e3) / 1e9 / float(peaks.get("hbm_gbs", 6650.0)), 4)}}


def run_e2e(god, torch, cfg, pattern, k, w, n_anchors, steps, dist, world, dev, inputs="host", device_out=None):
    href = torch.from_numpy(cfg.ref).pin_memory()
    hroff = torch.from_numpy(cfg.ref_offsets).pin_memory()
    hreads = torch.from_numpy(cfg.reads.seq).pin_memory()
    hroffs = torch.from_numpy(cfg.reads.offsets).pin_memory()
    n = cfg.reads.n
    n_anchors = int(n_anchors * 1.02) + 1024  # slack; the path is deterministic
    # god_anchor_compact (8 B: ref_pos, read_pos | strand << 31; the read id is implied by the anchor
    # offsets): the same result as god_seed_reads' 16-B anchors at half the D2H bytes
    an_host = torch.empty(n_anchors * 2 + 2, dtype=torch.uint32).pin_memory()
    ao_host = torch.empty(n + 1, dtype=torch.uint64).pin_memory()
    ph_host = torch.empty(max(1, n), dtype=torch.uint8).pin_memory()
    import ctypes
    from paper_2211_08157_b200 import _lib
    L = _lib.load()
    prm = _lib.GodParams(pattern.encode(), k, w)
    cut = _lib.GodCutoff(0, cfg.cutoff[0], cfg.cutoff[1], 0)
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    need = ctypes.c_uint64(0)
    vp = ctypes.c_void_p

    if inputs == "staged":
        dref = torch.empty_like(href, device=dev)
        droff = torch.empty_like(hroff, device=dev)
        dreads = torch.empty_like(hreads, device=dev)
        droffs = torch.empty_like(hroffs, device=dev)
    side = torch.cuda.Stream()
    main = torch.cuda.current_stream()

    def one_staged():
        # (--e2e-inputs staged) the caller stages the inputs itself: the reference in first (the index
        # needs all of it); the reads follow on a copy stream while the index is built; the seeding then
        # streams each read batch's results back to host buffers while later batches are seeded
        dref.copy_(href, non_blocking=True)
        droff.copy_(hroff, non_blocking=True)
        ref_in = torch.cuda.Event()
        ref_in.record(main)
        side.wait_event(ref_in)
        with torch.cuda.stream(side):
            dreads.copy_(hreads, non_blocking=True)
            droffs.copy_(hroffs, non_blocking=True)
        h = ctypes.c_void_p(0)
        _lib.check(L.god_build_index(ctypes.byref(prm), vp(dref.data_ptr()), vp(droff.data_ptr()), 1,
                                     ctypes.byref(cut), ctypes.byref(h), stream))
        main.wait_stream(side)
        _lib.check(L.god_seed_reads_compact(h, vp(dreads.data_ptr()), vp(droffs.data_ptr()), n, _lib.PHASE_SELECT,
                                    vp(ph_host.data_ptr()), 16, vp(an_host.data_ptr()), vp(ao_host.data_ptr()),
                                    n_anchors, ctypes.byref(need), stream))
        return h

    def one_host():
        # (default) every buffer handed to the C ABI is a pinned HOST buffer, one call:
        # god_build_index_and_seed streams the reference up in chunks with K1 running on the tiles that
        # are in, queues the first read batches right behind it (the link stays busy while the index is
        # sorted) and pipelines the read batches (H2D ahead, seeding, D2H of the 8-B anchors behind)
        h = ctypes.c_void_p(0)
        _lib.check(L.god_build_index_and_seed(ctypes.byref(prm), vp(href.data_ptr()), vp(hroff.data_ptr()), 1,
                                              ctypes.byref(cut), ctypes.byref(h), vp(hreads.data_ptr()),
                                              vp(hroffs.data_ptr()), n, _lib.PHASE_SELECT, vp(ph_host.data_ptr()), 16, 1,
                                              vp(an_host.data_ptr()), vp(ao_host.data_ptr()), n_anchors,
                                              ctypes.byref(need), stream))
        return h

    def one_host2():
        # (--e2e-inputs host2) the same buffers through the two separate calls
        h = ctypes.c_void_p(0)
        _lib.check(L.god_build_index(ctypes.byref(prm), vp(href.data_ptr()), vp(hroff.data_ptr()), 1,
                                     ctypes.byref(cut), ctypes.byref(h), stream))
        _lib.check(L.god_seed_reads_compact(h, vp(hreads.data_ptr()), vp(hroffs.data_ptr()), n, _lib.PHASE_SELECT,
                                    vp(ph_host.data_ptr()), 16, vp(an_host.data_ptr()), vp(ao_host.data_ptr()),
                                    n_anchors, ctypes.byref(need), stream))
        return h

    one = {"staged": one_staged, "host": one_host, "host2": one_host2}[inputs]

    L.god_index_free(one())  # warm-up
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    walls = []
    for _ in range(steps):
        t0 = time.perf_counter()
        L.god_index_free(one())
        walls.append(round((time.perf_counter() - t0) * 1e3, 1))
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    log(f"e2e wall ms per step: {walls}")
    ms = max_over_ranks(ms, dist, dev)
    h2d = cfg.ref.size + cfg.ref_offsets.nbytes + cfg.reads.seq.size + cfg.reads.offsets.nbytes
    d2h = int(need.value) * 8 + (n + 1) * 8 + n
    # the host results of the last e2e step against the device-resident step's (untimed): same phases, same
    # offsets, and every 8-B anchor = (ref_pos, read_pos | strand << 31) of the 16-B one, in the same order
    same = None
    if device_out and "an" in device_out:
        try:
            na = int(need.value)
            dan, dao, dph = device_out["an"], device_out["ao"], device_out["ph"]
            same = bool(int(dao.cpu()[n]) == na)
            if same:
                hc = an_host[: 2 * na].view(-1, 2).to(dev).to(torch.int64)
                da = dan[:na].to(torch.int64)
                same = bool(torch.equal(hc[:, 0], da[:, 0]) and torch.equal(hc[:, 1], da[:, 1] | (da[:, 3] << 31))
                            and torch.equal(ao_host.to(dev).view(torch.int64), dao.view(torch.int64))
                            and torch.equal(ph_host[:n].to(dev), dph[:n]))
                del hc, da
        except Exception as exc:  # never lose the bench line to the check itself
            log(f"e2e result check did not run: {exc!r}")
        log(f"e2e results equal the device-resident step's: {same}")
    return {"value": round(world * n / (ms / steps / 1e3), 1), "unit": "reads/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": steps, "ms_per_step": round(ms / steps, 3), "inputs": inputs,
            "equals_device_step": same,
            "outputs": "phases u8[n], anchor_offsets u64[n+1], god_anchor_compact[n_anchors] (8 B)"}


def run_reference(args, world, rank):
    """--impl reference: the CPU oracle, as it stands, on bounded samples of the same workload."""
    if world > 1 and rank != 0:
        return
    cfg, pattern, k, w = make_inputs(args.workload, args.scale, 0)
    times = []
    desc = ""
    spent = 0.0
    sbp = max(1_000_000, int(4_000_000 * args.scale))
    srd = max(500, int(4_000 * args.scale))
    ostages = None
    for i in range(args.warmup + args.steps):
        full_s, desc, sp, ostages = oracle_sample(cfg, pattern, k, w, sbp, srd)
        if i >= args.warmup:
            times.append(full_s)
            spent += sp
    full = float(np.mean(times))
    v = cfg.reads.n / full
    out = {"impl": "reference", "metric": METRIC, "value": round(v, 2), "unit": "reads/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(full * 1e3, 1), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
           "config": workload_config(args, cfg, pattern, k, w, world),
           "cpu_baseline": {"value": round(v, 2), "unit": "reads/s", "cores": 1, "kind": "oracle", "sample": desc,
                            "stages": ostages},
           "e2e": {"value": round(v, 2), "unit": "reads/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
