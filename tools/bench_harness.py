"""Seed-comparison harness benchmark (Fig. 4): N pairs of 1000-base
sequences with 0..300 substitutions per configuration of P:85, the GPU harness (seeds + rates +
Levenshtein) timed with CUDA events, accepted pairs at edit thresholds 20 / 138 / 295, and the CPU
oracle on a 1/100 sample.  usage: python tools/bench_harness.py [n_pairs] [iters]"""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (bounded CPU baseline only)
import paper_2211_08157_b200 as god  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
o, m, off, subs = synth.mutation_pairs(n, 1000, 300, 2024)
do, dm, doff = (torch.from_numpy(a).cuda() for a in (o, m, off))
E = torch.tensor([20, 138, 295], dtype=torch.uint64, device="cuda")
out = {"workload": f"{n} pairs x 1000 bases, 0..300 uniform substitutions (P:85)", "configs": {}}
for k, w, pat in [(8, 6, "110"), (8, 6, "10"), (8, 6, "101001"), (8, 6, "100"), (13, 9, "1110110110111"),
                  (18, 12, "111001011001010111"), (21, 11, "10"), (21, 11, "111101101101011101111")]:
    god.god_seed_harness(do, dm, doff, pat, k, w)
    torch.cuda.synchronize()
    god.profile_reset(); god.profile_enable(True)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        ed, mm, tt, ph = god.god_seed_harness(do, dm, doff, pat, k, w)
    e.record(); torch.cuda.synchronize()
    prof = god.profile_query(); god.profile_enable(False)
    ms = s.elapsed_time(e) / iters
    acc = god.god_harness_accepted(ed, mm, tt, E).cpu().numpy()
    ns = max(1, n // 100)
    t0 = time.perf_counter()
    oracle.harness_pairs(o[: ns * 1000], m[: ns * 1000], off[: ns + 1], k, w, pat)
    t_or = time.perf_counter() - t0
    key = f"k{k}-w{w}-{pat}"
    out["configs"][key] = {"ms": round(ms, 3), "pairs_per_s": round(n / (ms / 1e3), 1),
                           "kernels_ms": {kk: round(v[0] / iters, 3) for kk, v in prof.items()},
                           "accepted_at_E20_138_295": {a: acc[:, i].tolist() for i, a in enumerate(oracle.ALGOS)},
                           "oracle_pairs_per_s_1core": round(ns / t_or, 1)}
    print(key, out["configs"][key], flush=True)
print(json.dumps(out), flush=True)
