mkdir -p gpurun_out/r02c
for cfg in "1:1536" "4:1536" "16:1536" "1:1408" "1:1664" "16:1408"; do
sm=${cfg%%:*}; t=${cfg#*:}
GOD_SEG_SAMPLE=$sm GOD_BIN_TARGET=$t GOD_DEBUG_BUCKETS=1 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench_s$sm_$t.json 2> gpurun_out/r02c/bench_s$sm_$t.err
grep "\[bins\]" gpurun_out/r02c/bench_s$sm_$t.err | tail -1
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench_s$sm_$t.json').read().strip().splitlines()[-1])
print('sample $sm target $t', d['ms_per_step'], d['stage_ms'], {k:v['ms_per_step'] for k,v in d['kernels'].items() if k in ('k_bin_build','k_bucket_sort_big','k_seg_hist','k_rs_scatter')})
PY
done
