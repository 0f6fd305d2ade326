mkdir -p gpurun_out/r02c
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02c/parity_y.log 2>&1; tail -1 gpurun_out/r02c/parity_y.log
for ns in 1 0; do
if [ $ns = 1 ]; then export GOD_SEED_NO_SPLIT=1; else unset GOD_SEED_NO_SPLIT; fi
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench_y$ns.json 2> gpurun_out/r02c/bench_y$ns.err
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench_y$ns.json').read().strip().splitlines()[-1])
print('no_split=$ns', d['ms_per_step'], d['stage_ms'], {k:v['ms_per_step'] for k,v in d['kernels'].items() if 'probe' in k or 'extract_phase' in k or 'anchor' in k})
PY
done
