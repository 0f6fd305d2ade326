mkdir -p gpurun_out/r02c
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "index or repeat or probe" > gpurun_out/r02c/parity_idx.log 2>&1; tail -1 gpurun_out/r02c/parity_idx.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench_m.json 2> gpurun_out/r02c/bench_m.err
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench_m.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['stage_ms'], {k:v['ms_per_step'] for k,v in d['kernels'].items() if k in ('k_rs_scatter','k_rs_hist','k_seg_assign','scan_sort_hist','k_bin_build','k_bucket_sort_big')})
PY
