import os, sys, time, numpy as np, torch
sys.path.insert(0, '.')
import synth, paper_2211_08157_b200 as god
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
cfg = synth.make_config('human', scale=scale)
dref, doff = torch.from_numpy(cfg.ref).cuda(), torch.from_numpy(cfg.ref_offsets).cuda()
dr, dro = torch.from_numpy(cfg.reads.seq).cuda(), torch.from_numpy(cfg.reads.offsets).cuda()
ix = god.god_build_index(dref, doff, '10', 21, 11)
for it in range(3):
    god.profile_reset(); god.profile_enable(True)
    an, ao, ph = god.god_seed_reads(ix, dr, dro)
    torch.cuda.synchronize()
    prof = god.profile_query(); god.profile_enable(False)
    if it == 2: print({k: round(v[0], 3) for k, v in prof.items()}, int(an.shape[0]), flush=True)
