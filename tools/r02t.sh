mkdir -p gpurun_out/r02c
for fu in 0 1; do
if [ $fu = 1 ]; then export GOD_X2_FORCE_UNORDERED=1; fi
timeout 900 python bench.py --workload hifi --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench_t_$fu.json 2> gpurun_out/r02c/bench_t_$fu.err
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench_t_$fu.json').read().strip().splitlines()[-1])
print('force_unordered $fu', d['ms_per_step'], {k:v['ms_per_step'] for k,v in d['kernels'].items() if 'extract' in k})
PY
done
unset GOD_X2_FORCE_UNORDERED
ncu --set full --import-source on --clock-control none -k regex:k_extract3 -s 2 -c 1 -o gpurun_out/k1_hifi python tools/perf_step.py 1.0 hifi 0 > gpurun_out/ncu_k1_hifi.log 2>&1; tail -2 gpurun_out/ncu_k1_hifi.log
