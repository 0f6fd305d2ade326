mkdir -p gpurun_out/r02c
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02c/parity_x.log 2>&1; tail -2 gpurun_out/r02c/parity_x.log
timeout 300 python tools/perf_k1.py 1.0 10 3 2>&1 | tail -1
GOD_X2_NO_SLOTS=1 timeout 300 python tools/perf_k1.py 1.0 10 3 2>&1 | tail -1
