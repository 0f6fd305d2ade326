# Streamed host reference (god_build_index) and the e2e line with host inputs: parity first, then both e2e modes.
set -x
mkdir -p gpurun_out/r02s
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "streamed or host" > gpurun_out/r02s/test.log 2>&1; tail -5 gpurun_out/r02s/test.log
GOD_CHECKED=1 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "streamed" > gpurun_out/r02s/test_checked.log 2>&1; tail -3 gpurun_out/r02s/test_checked.log
python bench.py --steps 3 --warmup 3 --e2e-steps 4 --no-cpu-baseline --no-vote --e2e-inputs host > gpurun_out/r02s/bench_host.json 2> gpurun_out/r02s/bench_host.err; tail -3 gpurun_out/r02s/bench_host.err
python bench.py --steps 3 --warmup 3 --e2e-steps 4 --no-cpu-baseline --no-vote --e2e-inputs staged > gpurun_out/r02s/bench_staged.json 2> gpurun_out/r02s/bench_staged.err; tail -3 gpurun_out/r02s/bench_staged.err
