mkdir -p gpurun_out/r02c
python -m pytest tests/test_gpu_parity.py tests/test_gpu_checked.py -q -x > gpurun_out/r02c/parity_j.log 2>&1; tail -1 gpurun_out/r02c/parity_j.log
GOD_DEBUG_BUCKETS=1 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench_j.json 2> gpurun_out/r02c/bench_j.err
grep "\[bins\]" gpurun_out/r02c/bench_j.err | tail -1
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench_j.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['stage_ms'], {k:v['ms_per_step'] for k,v in d['kernels'].items() if v['ms_per_step']>0.2})
PY
