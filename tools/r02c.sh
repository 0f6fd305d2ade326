set -x
mkdir -p gpurun_out/r02c
python -m pytest tests/test_gpu_parity.py tests/test_gpu_checked.py tests/test_gpu_contain.py tests/test_gpu_vote.py -q -x > gpurun_out/r02c/parity.log 2>&1; tail -3 gpurun_out/r02c/parity.log
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench.json 2> gpurun_out/r02c/bench.err
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['stage_ms'], {k:v['ms_per_step'] for k,v in d['kernels'].items() if v['ms_per_step']>0.3})
PY
