#!/bin/bash
# k_post_sample resident blocks per SM (GC_PS_BLOCKS 6 vs 8) on the headline step
out=gpurun_out/r3i
mkdir -p $out
for r in 1 2 3; do
  for v in s6 s8; do
    GC_LIB_VARIANT=$v timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 0 > $out/${v}_$r.json 2> $out/${v}_$r.err
  done
done
GC_LIB_VARIANT=s6 timeout 300 python profiles/timeline.py plan24:kout+rem_cas+halve+splice 3 > $out/tl_s6.txt 2>&1
GC_LIB_VARIANT=s8 timeout 300 python profiles/timeline.py plan24:kout+rem_cas+halve+splice 3 > $out/tl_s8.txt 2>&1
