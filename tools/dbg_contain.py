import sys; sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np, torch, synth, paper_2211_08157_b200 as god
from test_gpu_contain import _contigs, _reads_from, cu
cs = _contigs(7); refs, ro = synth.concat(cs)
reads, qo = _reads_from(cs, [0, 1, 5, 12, 13, 30], 50, 60, length=150, p_sub=0.002, p_ins=0.0005, p_del=0.0005)
print("refs", refs.size, "reads", qo.size - 1, flush=True)
r = god.god_contain(cu(refs), cu(ro), cu(reads), cu(qo), "10", 21, 11, min_reads=20, cov=(1, 10))
print([x.cpu().numpy().sum() for x in r])
