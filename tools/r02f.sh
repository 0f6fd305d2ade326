mkdir -p gpurun_out/r02c
for v in rg16 mb6 mb8 rg16mb6; do
export GOD_LIB_VARIANT=$v
python -m pytest tests/test_gpu_parity.py -q -x -k "seed" > gpurun_out/r02c/parity_seed_$v.log 2>&1; tail -1 gpurun_out/r02c/parity_seed_$v.log
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench_$v.json 2> gpurun_out/r02c/bench_$v.err
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench_$v.json').read().strip().splitlines()[-1])
print('$v', d['ms_per_step'], d['stage_ms'], {k:v['ms_per_step'] for k,v in d['kernels'].items() if 'anchor' in k})
PY
done
