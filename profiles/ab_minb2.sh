#!/bin/bash
# giant-filter lock-step kernel: min-blocks 5 / 6 / 8 after the pass-through probe was dropped
out=gpurun_out/r3f
mkdir -p $out
for r in 1 2; do
  for v in g5 g6 g8; do GC_LIB_VARIANT=$v timeout 300 python profiles/incr_giant_probe.py > $out/${v}_$r.json 2>&1; done
done
timeout 600 python -m pytest tests/test_gpu_incremental.py tests/test_gpu_configs.py tests/test_gpu_knobs.py -m gpu -q -p no:cacheprovider > $out/tests.txt 2>&1; echo "tests rc=$?" >> $out/status.txt
