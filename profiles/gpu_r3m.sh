#!/bin/bash
# giant-filter clear folded into the probe kernel: incremental GPU suites + config-4 stream times
out=gpurun_out/r3m
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_incremental.py tests/test_gpu_configs.py tests/test_gpu_knobs.py tests/test_gpu_comm.py -m gpu -q -p no:cacheprovider > $out/tests.txt 2>&1; echo "tests rc=$?" >> $out/status.txt
for r in 1 2 3; do timeout 300 python profiles/incr_giant_probe.py > $out/g1_$r.json 2>&1; done
timeout 2400 python bench_configs.py --configs 4 --out $out/configs4.jsonl > $out/configs4.log 2>&1; echo "configs4 rc=$?" >> $out/status.txt
