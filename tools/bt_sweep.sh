for bt in 2048 2560 3072 3584; do echo "BT=$bt"; GOD_BIN_TARGET=$bt GOD_DEBUG_BUCKETS=1 python tools/perf_index.py 1.0 2>&1 | tail -3; done
