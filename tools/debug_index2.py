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
pattern, k, w, cut = '10', 15, 10, (1, 200)
os.makedirs('gpurun_out/dbg', exist_ok=True)
os.environ['GOD_DEBUG_DIR'] = 'gpurun_out/dbg'
ix = god.god_build_index(torch.from_numpy(ref).cuda(), torch.from_numpy(offs).cuda(), pattern, k, w, cutoff=cut)
print(ix.stats())
d = 'gpurun_out/dbg/'
L = lambda n, t: np.fromfile(d + n + '.bin', t)
hz = L('sorted_hz', np.uint64) & np.uint64((1 << 63) - 1)
print('sorted?', bool(np.all(np.diff(hz.astype(np.int64)) >= 0)))
rec = L('rec_hz', np.uint64) & np.uint64((1 << 63) - 1)
print('same multiset', np.array_equal(np.sort(rec), hz))
flag = L('flag', np.uint32); dix = L('dix', np.uint64); dstart = L('dstart', np.uint64); count = L('count', np.uint32)
kept = L('kept_off', np.uint64); kslot = L('kslot', np.uint32)
print('nd', flag.sum(), 'dix ok', np.array_equal(dix, np.concatenate([[0], np.cumsum(flag)[:-1]])))
heads = np.nonzero(flag)[0]
print('dstart ok', np.array_equal(dstart[:-1], heads), dstart[-1], hz.size)
print('count ok', np.array_equal(count, np.diff(dstart)))
st = ix.stats(); tau = st['tau']
kv = np.where(count <= tau, count, 0).astype(np.uint64)
print('kept_off ok', np.array_equal(kept[:count.size], np.concatenate([[0], np.cumsum(kv)[:-1]])))
print('kslot monotone', bool(np.all(np.diff(kslot.astype(np.int64)) >= 0)), kslot[:10], kslot[-10:])
