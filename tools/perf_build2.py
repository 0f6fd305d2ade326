"""Wall time of god_build_index vs the sum of its kernels, step by step (host-side gaps: allocation, syncs).
usage: python tools/perf_build2.py [workload] [steps]"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_2211_08157_b200 as god
wl = sys.argv[1] if len(sys.argv) > 1 else "human-1110"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
cfg, pattern, k, w = bench.make_inputs(wl, 1.0, 0)
dref, droff = torch.from_numpy(cfg.ref).cuda(), torch.from_numpy(cfg.ref_offsets).cuda()
for it in range(steps):
    god.profile_reset(); god.profile_enable(True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ix = god.god_build_index(dref, droff, pattern, k, w, cutoff=cfg.cutoff)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    prof = god.profile_query(); god.profile_enable(False)
    ks = sum(v[0] for v in prof.values())
    free, total = torch.cuda.mem_get_info()
    print(f"step {it}: wall {1e3*(t1-t0):.2f} ms, kernels {ks:.2f} ms, gap {1e3*(t1-t0)-ks:.2f} ms, free {free/1e9:.1f} GB", flush=True)
    ix.free()
