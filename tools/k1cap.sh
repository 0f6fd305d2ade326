# K1 check + capture on the GPU box: parity of the specialised kernel, timing, ncu source-level capture.
set -x
python -m pytest tests/test_gpu_parity.py -q -x -k "x2" > gpurun_out/k1_parity.log 2>&1; tail -3 gpurun_out/k1_parity.log
GOD_X2_DBG=0 python tools/perf_k1.py 1.0 10 3 > gpurun_out/perf_k1.log 2>&1; cat gpurun_out/perf_k1.log
GOD_X2_ANY_ORDER_TIMING=1 python tools/perf_k1.py 1.0 10 3 >> gpurun_out/perf_k1.log 2>&1; tail -1 gpurun_out/perf_k1.log
GOD_X2_ANY_ORDER_TIMING=1 ncu --set full --import-source on --clock-control none -k regex:k_extract -c 1 -o gpurun_out/k1_src python tools/perf_k1.py 0.25 10 1 > gpurun_out/ncu_k1.log 2>&1
tail -2 gpurun_out/ncu_k1.log
