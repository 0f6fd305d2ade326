mkdir -p gpurun_out/r02c
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_checked.py tests/test_gpu_contain.py -q -x > gpurun_out/r02c/parity_u.log 2>&1; tail -2 gpurun_out/r02c/parity_u.log
for wl in hifi ont hifi-110; do
timeout 600 python bench.py --workload $wl --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench_u_$wl.json 2> gpurun_out/r02c/bench_u_$wl.err
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench_u_$wl.json').read().strip().splitlines()[-1])
print('$wl', d['ms_per_step'], d['stage_ms'], {k:v['ms_per_step'] for k,v in d['kernels'].items() if 'extract' in k or 'x2' in k})
PY
done
