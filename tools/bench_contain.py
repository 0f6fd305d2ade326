"""Desk-scale containment search benchmark (Fig. 6).

Workload (synthetic stand-in for the paper's RefSeq / human / Pinus Taeda databases and wgsim
reads, none of which is in the container): a RefSeq-like database of N contigs with lognormal
lengths (i.i.d. bases, 3% of contigs carry a copy of a segment of another contig), reads simulated
from 10% of the contigs (the planted truth), the paper's k = 19, w = 16 and pattern sweep
('1' = no sparsification, '1110', '110', '10', '100'), reference batches of I bases ("-I").
Reports per pattern: GPU time of god_contain (index build of every batch + phase selection + seeding
+ voting + accumulation; inputs resident in HBM), accepted / planted / false accepts, the CPU
oracle on a bounded sample (one batch's worth of contigs and 1/20 of the reads), and prints one JSON
line.  usage: python tools/bench_contain.py [n_contigs] [n_reads] [iters]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (bounded CPU baseline only)
import paper_2211_08157_b200 as god  # noqa: E402
import synth  # noqa: E402

n_contigs = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
n_reads = int(sys.argv[2]) if len(sys.argv) > 2 else 200_000
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
K, W, I = 19, 16, 50_000_000
rng = np.random.default_rng(901)
lens = np.clip(rng.lognormal(np.log(40_000), 0.8, n_contigs).astype(np.int64), 2_000, 1_000_000)
contigs = [synth.iid_genome(int(L), 90_000 + i) for i, L in enumerate(lens)]
for i in rng.choice(n_contigs, n_contigs * 3 // 100, replace=False):
    j = int(rng.integers(0, n_contigs))
    L = int(min(5_000, contigs[i].size // 2, contigs[j].size))
    contigs[i][:L] = contigs[j][:L]
refs, ro = synth.concat(contigs)
present = np.sort(rng.choice(n_contigs, n_contigs // 10, replace=False))
per = max(1, n_reads // len(present))
seqs = []
for q, i in enumerate(present):
    rd = synth.simulate_reads(contigs[i], per, 5000 + q, length=150, start_margin=160, p_sub=0.001, p_ins=0.00005,
                              p_del=0.00005)
    seqs += [rd.seq[int(rd.offsets[x]):int(rd.offsets[x + 1])] for x in range(rd.n)]
reads, qo = synth.concat(seqs)
dref, dro, dq, dqo = (torch.from_numpy(a).cuda() for a in (refs, ro, reads, qo))
out = {"workload": f"desk containment: {n_contigs} contigs ({refs.size/1e6:.1f} Mbp, lognormal lengths), "
                   f"{qo.size - 1} x 150 bp reads from {len(present)} planted contigs, k={K}, w={W}, I={I} bases",
       "ref_bp": int(refs.size), "n_reads": int(qo.size - 1), "patterns": {}}
min_reads, cov = max(1, per // 4), (1, 20)
for pat in ["1", "1110", "110", "10", "100"]:
    kw = dict(batch_bases=I, min_reads=min_reads, cov=cov)
    god.god_contain(dref, dro, dq, dqo, pat, K, W, **kw)  # warm-up
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        mr, mb, acc = god.god_contain(dref, dro, dq, dqo, pat, K, W, **kw)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    acc = acc.cpu().numpy().astype(bool)
    truth = np.zeros(n_contigs, bool)
    truth[present] = True
    # bounded CPU oracle sample: the contigs of the first batch-sized prefix / 20, 1/20 of the reads
    nb = int(np.searchsorted(ro, I // 20, side="right")) - 1
    nb = max(1, min(nb, n_contigs))
    sub_ro = ro[:nb + 1].copy()
    sub_reads, sub_qo = synth.concat(seqs[: max(1, (qo.size - 1) // 20)])
    t0 = time.perf_counter()
    oracle.contain(refs[: int(sub_ro[-1])], sub_ro, sub_reads, sub_qo, pat, K, W, **kw)
    t_or = time.perf_counter() - t0
    out["patterns"][pat] = {"ms": round(ms, 2), "reads_per_s": round((qo.size - 1) / (ms / 1e3), 1),
                            "ref_gbp_per_s": round(refs.size / (ms / 1e3) / 1e9, 2),
                            "accepted": int(acc.sum()), "true_accepts": int((acc & truth).sum()),
                            "false_accepts": int((acc & ~truth).sum()), "planted": int(truth.sum()),
                            "oracle_sample_s": round(t_or, 2),
                            "oracle_sample": f"{nb} contigs ({int(sub_ro[-1])/1e6:.1f} Mbp), {sub_qo.size - 1} reads, 1 core"}
    print(pat, out["patterns"][pat], flush=True)
print(json.dumps(out), flush=True)
