set -x
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
( time python -m pytest tests -m gpu -q -x ) > gpurun_out/r02a/gputest.log 2>&1; tail -5 gpurun_out/r02a/gputest.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r02a/bench.json 2> gpurun_out/r02a/bench.err; tail -c 600 gpurun_out/r02a/bench.json
