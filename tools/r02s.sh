mkdir -p gpurun_out/r02c
for wl in hifi ont; do
timeout 900 python bench.py --workload $wl --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench_s_$wl.json 2> gpurun_out/r02c/bench_s_$wl.err
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench_s_$wl.json').read().strip().splitlines()[-1])
tot=sum(v['ms_per_step'] for v in d['kernels'].values())
print('$wl', d['ms_per_step'], d['stage_ms'], 'sum kernels', round(tot,2), 'anchors', d['n_anchors_per_step'])
for k,v in sorted(d['kernels'].items(), key=lambda kv:-kv[1]['ms_per_step'])[:12]: print(f"   {k:22s} {v['ms_per_step']:.4f} x{v['launches_per_step']}")
PY
done
