# Round-2 ncu --set full capture of the step's top kernels (human scale): K1 on the reference and on the
# reads, both LSD scatters, k_bin_build, the probe and the anchor writer.  After the program has run
# cleanly without ncu (tools/r02final.sh).
set -x
mkdir -p gpurun_out/r02
ncu --set full --import-source on --clock-control none -k "regex:k_extract3|k_bin_build|k_rs_scatter2|k_anchor_count|k_anchor_write1" -c 7 -o gpurun_out/r02/full_top python tools/perf_step.py 1.0 human 0 > gpurun_out/r02/ncu_full.log 2>&1; tail -2 gpurun_out/r02/ncu_full.log
