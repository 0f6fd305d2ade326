mkdir -p gpurun_out/r02c
export GOD_LIB_VARIANT=
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02c/bench_noent.json 2> gpurun_out/r02c/bench_noent.err
python - <<PY
import json
d=json.loads(open('gpurun_out/r02c/bench_noent.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['stage_ms'], {k:v['ms_per_step'] for k,v in d['kernels'].items() if v['ms_per_step']>0.3})
PY
unset GOD_LIB_VARIANT
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,smsp__inst_executed.sum --clock-control none -k "regex:k_anchor_write|k_anchor_count" --csv --log-file gpurun_out/r02c/ncu_seed.csv python tools/perf_step.py 1.0 human 0 > /dev/null 2>&1
grep -E "k_anchor" gpurun_out/r02c/ncu_seed.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-200
