"""Time god_vote_reads per kernel on a BASELINE config (python tools/perf_vote.py [workload] [scale])."""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_2211_08157_b200 as god
W = {"human": ("human", "10", 21, 11), "illumina": ("illumina", "10", 21, 11), "hifi": ("hifi", "10", 19, 19),
     "ont": ("ont", "10", 15, 10), "tiny": ("tiny", "10", 21, 11)}
name = sys.argv[1] if len(sys.argv) > 1 else "human"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
c, pat, k, w = W[name]
cfg = synth.make_config(c, scale=scale)
dref, doff = torch.from_numpy(cfg.ref).cuda(), torch.from_numpy(cfg.ref_offsets).cuda()
dr, dro = torch.from_numpy(cfg.reads.seq).cuda(), torch.from_numpy(cfg.reads.offsets).cuda()
ix = god.god_build_index(dref, doff, pat, k, w, cutoff=cfg.cutoff)
an, ao, ph = god.god_seed_reads(ix, dr, dro)
per = np.diff(ao.cpu().numpy())
res = {"workload": name, "n_reads": cfg.reads.n, "n_anchors": int(an.shape[0]),
       "reads_by_class": [int(((per > 0) & (per <= 32)).sum()), int(((per > 32) & (per <= 2048)).sum()),
                          int((per > 2048).sum())], "max_anchors_per_read": int(per.max())}
for it in range(4):
    god.profile_reset(); god.profile_enable(True)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    v, vo = god.god_vote_reads(ix, dr, dro, ph, an, ao, D=0, V=3, max_pairs=0)
    e.record(); torch.cuda.synchronize()
    prof = god.profile_query(); god.profile_enable(False)
    if it == 3:
        vv = god.votes_numpy(v)
        res.update({"vote_ms": round(s.elapsed_time(e), 3), "kernels_ms": {kk: round(x[0], 3) for kk, x in prof.items()},
                    "n_votes": int(vv.size), "rescued": int(vv["rescued"].sum())})
print(json.dumps(res), flush=True)
