mkdir -p gpurun_out/r02c
GOD_DEBUG_BUCKETS=1 timeout 900 python bench.py --workload human-1110 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench_p.json 2> gpurun_out/r02c/bench_p.err
grep "\[bins\]" gpurun_out/r02c/bench_p.err | tail -2
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench_p.json').read().strip().splitlines()[-1])
tot=sum(v['ms_per_step'] for v in d['kernels'].values())
print(d['ms_per_step'], d['stage_ms'], 'sum kernels', tot)
for k,v in sorted(d['kernels'].items(), key=lambda kv:-kv[1]['ms_per_step'])[:14]: print(f"{k:22s} {v['ms_per_step']:.4f} x{v['launches_per_step']}")
PY
