"""How much would overlapping the index build with the seeding of another batch gain?  Two host threads,
two streams: thread A builds the index of the reference (device buffers), thread B seeds the reads against
an index built before.  Wall time of both together against the sum of each alone (a bound on what a
pipelined server, or a K1-over-reads hoisted beside the index sort, could gain)."""
import sys, threading, time
sys.path.insert(0, '.')
import torch
import bench
import paper_2211_08157_b200 as god
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
cfg, pattern, k, w = bench.make_inputs('human', scale, 0)
dref = torch.from_numpy(cfg.ref).cuda(); droff = torch.from_numpy(cfg.ref_offsets).cuda()
dreads = torch.from_numpy(cfg.reads.seq).cuda(); droffs = torch.from_numpy(cfg.reads.offsets).cuda()
ix0 = god.god_build_index(dref, droff, pattern, k, w, cutoff=cfg.cutoff)
an, ao, ph = god.god_seed_reads(ix0, dreads, droffs)
cap = int(an.shape[0]); n = cfg.reads.n
out = (torch.empty((cap, 4), dtype=torch.uint32, device='cuda'), torch.empty(n + 1, dtype=torch.uint64, device='cuda'),
       torch.empty(n, dtype=torch.uint8, device='cuda'))
del an
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
def build():
    with torch.cuda.stream(sa):
        ix = god.god_build_index(dref, droff, pattern, k, w, cutoff=cfg.cutoff)
        sa.synchronize(); ix.free()
def seed():
    with torch.cuda.stream(sb):
        god.god_seed_reads(ix0, dreads, droffs, cap=cap, out=out)
        sb.synchronize()
def timed(fns, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        th = [threading.Thread(target=f) for f in fns]
        [t.start() for t in th]; [t.join() for t in th]
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    return best * 1e3
for _ in range(2):
    build(); seed()
b, s, both = timed([build]), timed([seed]), timed([build, seed])
print(f"build alone {b:.1f} ms, seed alone {s:.1f} ms, sum {b + s:.1f} ms, both concurrently {both:.1f} ms", flush=True)
