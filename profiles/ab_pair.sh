#!/bin/bash
# Rem-CAS row pairing (GC_ROW_PAIR) A/B on the headline step, plus the union-find GPU suites on the default build
out=gpurun_out/r3h
mkdir -p $out
for r in 1 2 3; do
  for v in p0 p1; do
    GC_LIB_VARIANT=$v timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 0 > $out/${v}_$r.json 2> $out/${v}_$r.err
  done
done
timeout 900 python -m pytest tests/test_gpu_static.py tests/test_gpu_stress.py tests/test_gpu_forest.py tests/test_gpu_knobs.py tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider > $out/tests.txt 2>&1; echo "tests rc=$?" >> $out/status.txt
