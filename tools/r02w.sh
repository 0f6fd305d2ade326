mkdir -p gpurun_out/r02c
for fm in 64 1000000; do
for wl in hifi ont; do
GOD_SEED_FAST_MAX=$fm timeout 600 python bench.py --workload $wl --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench_w_$wl.json 2> gpurun_out/r02c/bench_w_$wl.err
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench_w_$wl.json').read().strip().splitlines()[-1])
print('fast_max $fm $wl', d['ms_per_step'], d['stage_ms'], {k:v['ms_per_step'] for k,v in d['kernels'].items() if v['ms_per_step']>0.25})
PY
done
done
