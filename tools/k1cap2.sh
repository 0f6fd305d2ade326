set -x
ncu --set full --import-source on --clock-control none -k regex:k_extract -c 1 -o gpurun_out/k1_src python tools/perf_index.py 0.25 > gpurun_out/ncu_k1.log 2>&1
tail -2 gpurun_out/ncu_k1.log
