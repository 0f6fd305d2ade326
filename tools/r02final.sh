# Round-2 measurement on the GPU box: GPU suite (all 9 whole-config digest rows), bench line, per-kernel
# ncu traffic of one step, launch list of the bench command, measurement table.
set -x
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
( time python -m pytest tests -m gpu -q ) > gpurun_out/r02/gputest_final.log 2>&1; tail -3 gpurun_out/r02/gputest_final.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r02/bench_final.json 2> gpurun_out/r02/bench_final.err; tail -c 300 gpurun_out/r02/bench_final.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum --clock-control none -o gpurun_out/r02/step_metrics python tools/perf_step.py 1.0 human 0 > gpurun_out/r02/ncu_step.log 2>&1; tail -2 gpurun_out/r02/ncu_step.log
python tools/ncu_step_traffic.py gpurun_out/r02/step_metrics.ncu-rep gpurun_out/r02/ncu_traffic_r02.json > gpurun_out/r02/traffic.txt 2>&1; tail -5 gpurun_out/r02/traffic.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02/ncu_launch.log 2>&1; tail -1 gpurun_out/r02/ncu_launch.log
python tools/measure_table.py gpurun_out/parity_digests.jsonl > gpurun_out/r02/table.md 2> gpurun_out/r02/table.err; tail -30 gpurun_out/r02/table.md
