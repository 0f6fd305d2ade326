mkdir -p gpurun_out/r02c
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "slotted or mixed or determin" > gpurun_out/r02c/parity_v.log 2>&1; tail -3 gpurun_out/r02c/parity_v.log
GOD_CHECKED=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "slotted" > gpurun_out/r02c/parity_vc.log 2>&1; tail -2 gpurun_out/r02c/parity_vc.log
