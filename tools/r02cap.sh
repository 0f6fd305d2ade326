# Round-2 measurement call on the GPU box: GPU suite, bench line, K1 compute floor, per-kernel traffic of
# one full step (ncu metrics pass), launch list of the bench command.
set -x
mkdir -p gpurun_out/r02
python -m pytest tests -m gpu -q > gpurun_out/r02/gputest.log 2>&1; tail -3 gpurun_out/r02/gputest.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r02/bench.json 2> gpurun_out/r02/bench.err; tail -c 400 gpurun_out/r02/bench.json
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/k1_floor tools/k1_floor.cu && ./tools/k1_floor > gpurun_out/r02/k1_floor.json; cat gpurun_out/r02/k1_floor.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum --clock-control none -o gpurun_out/r02/step_metrics python tools/perf_step.py 1.0 human 0 > gpurun_out/r02/ncu_step.log 2>&1; tail -2 gpurun_out/r02/ncu_step.log
python tools/ncu_step_traffic.py gpurun_out/r02/step_metrics.ncu-rep profiles/ncu_traffic_r02.json > gpurun_out/r02/traffic.txt 2>&1; cp profiles/ncu_traffic_r02.json gpurun_out/r02/; cat gpurun_out/r02/traffic.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-vote > gpurun_out/r02/ncu_launch.log 2>&1; tail -1 gpurun_out/r02/ncu_launch.log
