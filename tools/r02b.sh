# Re-entry check on the GPU box: GPU suite on HEAD, bench line, pipe microbenchmark.
set -x
mkdir -p gpurun_out/r02b
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
( time python -m pytest tests -m gpu -q -x ) > gpurun_out/r02b/gputest.log 2>&1; tail -5 gpurun_out/r02b/gputest.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r02b/bench.json 2> gpurun_out/r02b/bench.err; tail -c 600 gpurun_out/r02b/bench.json
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_microbench tools/pipe_microbench.cu && ./tools/pipe_microbench > gpurun_out/r02b/pipe.jsonl; cat gpurun_out/r02b/pipe.jsonl
