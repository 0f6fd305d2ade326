import os, sys, time, numpy as np, torch
sys.path.insert(0, '.')
import synth, paper_2211_08157_b200 as god
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.2
ref = synth.reference_for('human', scale)
off = np.array([0, ref.size], np.uint64)
dref, doff = torch.from_numpy(ref).cuda(), torch.from_numpy(off).cuda()
for flags in ["0", "2", "1", "3"]:
    os.environ["GOD_X2_DBG"] = flags
    for it in range(3):
        god.profile_reset(); god.profile_enable(True)
        h = god.god_minimizers(dref, doff, '10', 21, 11, global_pos=True)
        torch.cuda.synchronize()
        prof = god.profile_query(); god.profile_enable(False)
        if it == 2: print("flags", flags, {k: round(v[0], 3) for k, v in prof.items() if 'extract' in k}, int(h[0].shape[0]), flush=True)
        del h
