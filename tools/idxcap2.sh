set -x
ncu --set full --import-source on --clock-control none -k "regex:k_rs_scatter|k_bin_build|k_seg_assign|k_anchor_write|k_anchor_count" -c 7 -o gpurun_out/idx_src python tools/perf_step.py 0.25 human 0 > gpurun_out/ncu_idx.log 2>&1
tail -2 gpurun_out/ncu_idx.log
