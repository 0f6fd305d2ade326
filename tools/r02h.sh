mkdir -p gpurun_out/r02c
for cfg in ":3072" "bs256:1536" "bs256:1792" "bs256:1920"; do
v=${cfg%%:*}; t=${cfg#*:}
export GOD_LIB_VARIANT=$v
if [ "$t" = "3072" -o "$t" = "1536" ]; then python -m pytest tests/test_gpu_parity.py -q -x -k "index or repeat or probe" > gpurun_out/r02c/parity_idx_$v.log 2>&1; tail -1 gpurun_out/r02c/parity_idx_$v.log; fi
GOD_BIN_TARGET=$t GOD_DEBUG_BUCKETS=1 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench_t$t.json 2> gpurun_out/r02c/bench_t$t.err
grep "\[bins\]" gpurun_out/r02c/bench_t$t.err | tail -1
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench_t$t.json').read().strip().splitlines()[-1])
print('$v $t', d['ms_per_step'], d['stage_ms'], {k:v['ms_per_step'] for k,v in d['kernels'].items() if k in ('k_bin_build','k_bucket_sort_big','k_big_dir','k_rs_scatter','k_probe','k_tau')})
PY
done
