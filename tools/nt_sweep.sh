set -x
mkdir -p gpurun_out/nt
for v in nt256; do
  export GOD_LIB_VARIANT=$v
  python -m pytest tests/test_gpu_parity.py -q -x -k "x2 or seed or minimizer" > gpurun_out/nt/parity_$v.log 2>&1; tail -2 gpurun_out/nt/parity_$v.log
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/nt/bench_$v.json 2> gpurun_out/nt/bench_$v.err
  python - <<PY
import json
d=json.loads(open('gpurun_out/nt/bench_$v.json').read().strip().splitlines()[-1])
print('$v', d['ms_per_step'], {k:v['ms_per_step'] for k,v in d['kernels'].items() if 'extract' in k or 'tile_desc' in k})
PY
done
