import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synth, oracle, paper_2211_08157_b200 as god
rng = np.random.default_rng(7)
rep = synth.random_acgt(rng, 700)
parts = []
for i in range(60):
    parts += [synth.random_acgt(rng, int(rng.integers(500, 5000)), 0.001), rep]
seqs = [np.concatenate(parts[i:i + 10]) for i in range(0, len(parts), 10)] + [np.zeros(0, np.uint8)]
ref, offs = synth.concat(seqs)
pattern, k, w, cut = '10', 15, 10, (1, 200)
dumps = []
for rep_i in range(3):
    ix = god.god_build_index(torch.from_numpy(ref).cuda(), torch.from_numpy(offs).cuda(), pattern, k, w, cutoff=cut)
    dumps.append(ix.dump()); st = ix.stats()
print('stats', st)
print('deterministic:', all(np.array_equal(dumps[0][i], d[i]) for d in dumps[1:] for i in range(3)))
ox = oracle.Index(ref, offs, pattern, k, w, cutoff=cut)
oh, op, oz = ox.dump()
h, p, z = dumps[0]
bad = np.nonzero(h != oh)[0]
print('n mismatch', bad.size, bad[:20])
for b in bad[:5]:
    lo, hi = max(0, b-3), b+4
    print('idx', b)
    for i in range(lo, hi):
        print(i, h[i], oh[i], h[i] >> 17, oh[i] >> 17, p[i], op[i], z[i], oz[i])
# check E multiset
E, _ = oracle.minimizers_batch(ref, offs, pattern, k, w, global_pos=True)
gh, gp, gz, go = god.god_minimizers(ref, offs, pattern, k, w, global_pos=True)
print('mz equal', np.array_equal(gh, E['hash']), np.array_equal(gp.astype(np.uint64), E['pos']))
