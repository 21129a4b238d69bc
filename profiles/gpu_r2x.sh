#!/bin/bash
# compute-sanitizer memcheck over the whole GPU test suite (round-2 code)
out=gpurun_out/r2x
mkdir -p $out
timeout 3300 compute-sanitizer --tool memcheck --print-limit 50 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > $out/memcheck_gpu_suite.txt 2>&1
echo "memcheck suite rc=$?" >> $out/status.txt
