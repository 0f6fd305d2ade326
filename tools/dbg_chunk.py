"""Localise a whole-config digest mismatch of the reference minimizers: GPU god_minimizers records
[lo, hi) (position order) against the oracle on the covering sub-sequence (phase-aligned start,
margins), first differing record with context.
usage: python tools/dbg_chunk.py CONFIG PATTERN LO HI"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2211_08157_b200 as god  # noqa: E402
import synth  # noqa: E402

cfgname, pat, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
cfg = synth.make_config(cfgname)
k, w = cfg.k, cfg.w
ref, roff = cfg.ref, cfg.ref_offsets
h, p, z, mo = god.god_minimizers(torch.from_numpy(ref).cuda(), torch.from_numpy(roff).cuda(), pat, k, w, global_pos=True)
gh, gp, gz = h[lo:hi].cpu().numpy(), p[lo:hi].cpu().numpy().astype(np.int64), z[lo:hi].cpu().numpy()
del h, p, z
print("gpu records", lo, hi, "pos", gp.min(), gp.max(), "sorted:", bool(np.all(np.diff(gp) > 0)), flush=True)
P = len(pat)
a = max(0, (int(gp.min()) - 20000) // P * P)
b = min(ref.size, int(gp.max()) + 20000)
sub = np.ascontiguousarray(ref[a:b])
om, oo = oracle.minimizers_batch(sub, np.array([0, sub.size], np.uint64), pat, k, w, global_pos=False)
op = om["pos"].astype(np.int64) + a
core = (op >= gp.min() + 2000) & (op <= gp.max() - 2000)
oh2, op2, oz2 = om["hash"][core], op[core], om["strand"][core]
gcore = (gp >= gp.min() + 2000) & (gp <= gp.max() - 2000)
gh2, gp2, gz2 = gh[gcore], gp[gcore], gz[gcore]
print("core records gpu", gh2.size, "oracle", oh2.size, flush=True)
n = min(gh2.size, oh2.size)
d = np.nonzero((gh2[:n] != oh2[:n]) | (gp2[:n] != op2[:n]) | (gz2[:n] != oz2[:n]))[0]
if d.size == 0 and gh2.size == oh2.size:
    print("core identical")
else:
    i = int(d[0]) if d.size else n
    print("first difference at core index", i)
    for j in range(max(0, i - 5), min(n, i + 8)):
        print(j, "gpu", int(gh2[j]), int(gp2[j]), int(gz2[j]), "| oracle", int(oh2[j]), int(op2[j]), int(oz2[j]))
    # the raw sequence around the position
    q = int(min(gp2[i] if i < gp2.size else op2[i], op2[i] if i < op2.size else gp2[i]))
    print("ref around", q, bytes(ref[q - 60:q + 60]).decode(errors="replace"))
