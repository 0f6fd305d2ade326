# Streamed host reference (god_build_index), the 4-slot seeding pipeline and god_build_index_and_seed:
# parity first (plain and checked builds), then the e2e line in its three input modes.
set -x
mkdir -p gpurun_out/r02s
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "streamed or host or compact or build_index_and_seed" > gpurun_out/r02s/test.log 2>&1; tail -5 gpurun_out/r02s/test.log
GOD_CHECKED=1 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "streamed or build_index_and_seed or pipelined" > gpurun_out/r02s/test_checked.log 2>&1; tail -3 gpurun_out/r02s/test_checked.log
for m in host host2 staged; do
GOD_PIPE_TRACE=1 python bench.py --steps 3 --warmup 3 --e2e-steps 4 --no-cpu-baseline --no-vote --e2e-inputs $m > gpurun_out/r02s/bench_$m.json 2> gpurun_out/r02s/bench_$m.err; tail -10 gpurun_out/r02s/bench_$m.err
done
