#!/bin/bash
# parent reads with an L2 evict_last hint (GC_P_HINT) on the headline step and at s26
out=gpurun_out/r3n
mkdir -p $out
for r in 1 2 3; do
  for v in h0 h1; do
    GC_LIB_VARIANT=$v timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 0 > $out/${v}_$r.json 2> $out/${v}_$r.err
  done
done
for v in h0 h1; do GC_LIB_VARIANT=$v timeout 600 python profiles/single_scale.py 25 26 > $out/${v}_scale.jsonl 2>&1; done
