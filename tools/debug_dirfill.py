import os, sys, numpy as np, torch, time
sys.path.insert(0, '.')
import synth, paper_2211_08157_b200 as god
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.2
ref = synth.reference_for('human', scale)
off = np.array([0, ref.size], np.uint64)
os.makedirs('/tmp/dbgdir', exist_ok=True)
os.environ['GOD_DEBUG_DIR'] = '/tmp/dbgdir'
os.environ['GOD_DISABLE_X2'] = '1'
ix = god.god_build_index(torch.from_numpy(ref).cuda(), torch.from_numpy(off).cuda(), '10', 21, 11)
st = ix.stats(); print(st)
ks = np.fromfile('/tmp/dbgdir/kslot.bin', np.uint32)
d = np.diff(ks.astype(np.int64))
print('kslot n', ks.size, 'first', ks[:5], 'last', ks[-5:], 'min diff', d.min(), 'max diff', d.max(), 'argmax', d.argmax())
dirr = np.fromfile('/tmp/dbgdir/dir.bin', np.uint32)
print('dir monotone', bool(np.all(np.diff(dirr.astype(np.int64)) >= 0)), dirr[:3], dirr[-3:])
god.profile_enable(True); god.profile_reset()
ix2 = god.god_build_index(torch.from_numpy(ref).cuda(), torch.from_numpy(off).cuda(), '10', 21, 11)
print({k: v for k, v in god.profile_query().items()})
