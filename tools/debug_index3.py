import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import synth, oracle, paper_2211_08157_b200 as god
rng = np.random.default_rng(7)
rep = synth.random_acgt(rng, 700)
parts = []
for i in range(60):
    parts += [synth.random_acgt(rng, int(rng.integers(500, 5000)), 0.001), rep]
seqs = [np.concatenate(parts[i:i + 10]) for i in range(0, len(parts), 10)] + [np.zeros(0, np.uint8)]
ref, offs = synth.concat(seqs)
pattern, k, w = '10', 15, 10
for cut in [(1, 5000), (1, 200), (1, 20)]:
    ox = oracle.Index(ref, offs, pattern, k, w, cutoff=cut)
    oh, op, oz = ox.dump()
    res = []
    keep = []
    for t in range(4):
        ix = god.god_build_index(torch.from_numpy(ref).cuda(), torch.from_numpy(offs).cuda(), pattern, k, w, cutoff=cut)
        keep.append(ix)
        dumps = [ix.dump() for _ in range(3)]
        dd = ix.dump(device=True)
        dev_ok = np.array_equal(dd[0].cpu().numpy(), oh)
        res.append((all(np.array_equal(dumps[0][0], d[0]) for d in dumps), [np.array_equal(d[0], oh) for d in dumps], dev_ok))
    print(cut, res)
