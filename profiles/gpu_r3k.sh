#!/bin/bash
out=gpurun_out/r3k
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_forest.py tests/test_gpu_configs.py tests/test_gpu_static.py -m gpu -q -p no:cacheprovider -x > $out/tests.txt 2>&1; echo "tests rc=$?" >> $out/status.txt
for r in 1 2; do timeout 300 python profiles/bfs_time.py 27 bfs+async+halve > $out/c5_$r.txt 2>&1; done
timeout 300 python profiles/timeline.py forest_uniform27 1 > $out/tl_forest27.txt 2>&1
