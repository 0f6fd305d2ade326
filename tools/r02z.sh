mkdir -p gpurun_out/r02c
for cfg in "1:1" "2:1" "2:2" "3:2"; do
export GOD_SPLIT_PROBE_CTAS=${cfg%%:*} GOD_SPLIT_LESS=${cfg#*:}
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench_z.json 2> gpurun_out/r02c/bench_z.err
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench_z.json').read().strip().splitlines()[-1])
print('probe_ctas:less=$cfg', d['ms_per_step'], d['stage_ms'], {k:v['ms_per_step'] for k,v in d['kernels'].items() if 'probe' in k or 'extract_phase' in k})
PY
done
