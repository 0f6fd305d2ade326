import os, sys, time, numpy as np, torch
sys.path.insert(0, '.')
import synth, paper_2211_08157_b200 as god
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
ref = synth.reference_for('human', scale)
off = np.array([0, ref.size], np.uint64)
dref, doff = torch.from_numpy(ref).cuda(), torch.from_numpy(off).cuda()
for it in range(3):
    god.profile_reset(); god.profile_enable(True)
    ix = god.god_build_index(dref, doff, '10', 21, 11)
    torch.cuda.synchronize()
    prof = god.profile_query(); god.profile_enable(False)
    st = ix.stats(); ix.free()
    if it == 2:
        print({k: round(v[0], 3) for k, v in prof.items()}, flush=True)
        print('total kernels', round(sum(v[0] for v in prof.values()), 2), st['n_distinct_all'], st['kept_entries'], flush=True)
