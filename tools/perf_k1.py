"""Time K1 (god_minimizers on the reference, the specialised kernel) at a given scale and pattern.
usage: python tools/perf_k1.py [scale] [pattern] [iters]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_2211_08157_b200 as god
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.2
pat = sys.argv[2] if len(sys.argv) > 2 else "10"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5
ref = synth.reference_for('human', scale)
off = np.array([0, ref.size], np.uint64)
dref, doff = torch.from_numpy(ref).cuda(), torch.from_numpy(off).cuda()
ts = []
for it in range(iters):
    god.profile_reset(); god.profile_enable(True)
    h = god.god_minimizers(dref, doff, pat, 21, 11, global_pos=True)
    torch.cuda.synchronize()
    prof = god.profile_query(); god.profile_enable(False)
    ts.append({k: round(v[0], 3) for k, v in prof.items() if 'extract' in k})
    n = int(h[0].shape[0]); del h
print("k1", pat, scale, ts[-1], "records", n, "positions", god.profile_units("extract_ref") or "-", flush=True)
