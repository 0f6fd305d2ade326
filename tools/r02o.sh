mkdir -p gpurun_out/r02c
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r02c/parity_o.log 2>&1; tail -1 gpurun_out/r02c/parity_o.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench_o.json 2> gpurun_out/r02c/bench_o.err
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench_o.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['stage_ms'], {k:v['ms_per_step'] for k,v in d['kernels'].items() if v['ms_per_step']>2})
PY
