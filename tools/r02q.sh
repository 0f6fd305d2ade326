python tools/perf_build2.py human-1110 6
GOD_SEG_SAMPLE=1 python tools/perf_build2.py human-1110 6
python tools/perf_build2.py human 4
