mkdir -p gpurun_out/r02c
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checked.py -q -x > gpurun_out/r02c/parity_l.log 2>&1; tail -2 gpurun_out/r02c/parity_l.log
for wl in human-1 human; do
GOD_DEBUG_BUCKETS=1 timeout 600 python bench.py --workload $wl --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench_l_$wl.json 2> gpurun_out/r02c/bench_l_$wl.err
grep "\[bins\]" gpurun_out/r02c/bench_l_$wl.err | tail -1
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench_l_$wl.json').read().strip().splitlines()[-1])
print('$wl', d['ms_per_step'], d['stage_ms'], {k:v['ms_per_step'] for k,v in d['kernels'].items() if v['ms_per_step']>0.5})
PY
done
