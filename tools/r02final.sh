# Round-2 final measurement: GPU suite (all 9 whole-config digest rows), bench line, measurement table.
set -x
mkdir -p gpurun_out/r02
python -m pytest tests -m gpu -q > gpurun_out/r02/gputest_final.log 2>&1; tail -3 gpurun_out/r02/gputest_final.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r02/bench_final.json 2> gpurun_out/r02/bench_final.err; tail -c 300 gpurun_out/r02/bench_final.json
python tools/measure_table.py gpurun_out/parity_digests.jsonl > gpurun_out/r02/table.md 2> gpurun_out/r02/table.err; cat gpurun_out/r02/table.md
