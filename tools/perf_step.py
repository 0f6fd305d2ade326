"""One hot-path step (index build + SELECT-mode seeding) of a BASELINE workload, for ncu captures.
usage: python tools/perf_step.py [scale] [workload] [warm]   (warm: untimed steps before the captured one)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2211_08157_b200 as god  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
wl = sys.argv[2] if len(sys.argv) > 2 else "human"
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg, pattern, k, w = bench.make_inputs(wl, scale, 0)
dref, droff = torch.from_numpy(cfg.ref).cuda(), torch.from_numpy(cfg.ref_offsets).cuda()
dreads, droffs = torch.from_numpy(cfg.reads.seq).cuda(), torch.from_numpy(cfg.reads.offsets).cuda()
for it in range(warm + 1):
    ix = god.god_build_index(dref, droff, pattern, k, w, cutoff=cfg.cutoff)
    an, ao, ph = god.god_seed_reads(ix, dreads, droffs)
    torch.cuda.synchronize()
    st = ix.stats()
    ix.free()
print("step", wl, scale, st["n_entries_all"], int(an.shape[0]), flush=True)
