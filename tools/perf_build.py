import os, sys, time, numpy as np, torch
sys.path.insert(0, '.')
import synth, paper_2211_08157_b200 as god
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
ref = synth.reference_for('human', scale)
off = np.array([0, ref.size], np.uint64)
dref, doff = torch.from_numpy(ref).cuda(), torch.from_numpy(off).cuda()
for mode in ("keep", "free"):
    keep = []
    for i in range(4):
        god.profile_reset(); god.profile_enable(True)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ix = god.god_build_index(dref, doff, '10', 21, 11)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        prof = god.profile_query(); god.profile_enable(False)
        ks = sum(v[0] for v in prof.values())
        print(mode, i, f"wall {1e3*(t1-t0):.1f} ms  kernels {ks:.1f} ms", flush=True)
        if mode == "keep": keep.append(ix)
        else: ix.free()
    for x in keep: x.free()
