mkdir -p gpurun_out/r02c
for wl in human-1110 human-110 human; do
timeout 900 python bench.py --workload $wl --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench_r_$wl.json 2> gpurun_out/r02c/bench_r_$wl.err
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench_r_$wl.json').read().strip().splitlines()[-1])
tot=sum(v['ms_per_step'] for v in d['kernels'].values())
print('$wl', d['ms_per_step'], d['stage_ms'], 'sum kernels', round(tot,2))
PY
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_contain.py -q -x > gpurun_out/r02c/parity_r.log 2>&1; tail -1 gpurun_out/r02c/parity_r.log
