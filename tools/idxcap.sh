# Index-build stage check on the GPU box: timings, bin statistics, ncu captures of the stage-3 kernels.
set -x
GOD_DEBUG_BUCKETS=1 python tools/perf_index.py 1.0 > gpurun_out/perf_index.log 2>&1; cat gpurun_out/perf_index.log
ncu --set full --import-source on --clock-control none -k "regex:k_rs_scatter|k_bin_build|k_bucket_sort_big|k_seg_assign" -c 5 -o gpurun_out/idx_src python tools/perf_index.py 0.25 > gpurun_out/ncu_idx.log 2>&1
tail -2 gpurun_out/ncu_idx.log
