#!/bin/bash
# A/B of k_union_coo_async_mlp's __launch_bounds__ min-blocks (occupancy vs
# spills) on the config-4 stream, filter on and off; variants from build_variants.sh
out=gpurun_out/r3c
mkdir -p $out
for r in 1 2; do
  for v in m55 m86 m88 m66; do
    GC_LIB_VARIANT=$v timeout 300 python profiles/incr_giant_probe.py > $out/${v}_g1_$r.json 2>&1
    GC_LIB_VARIANT=$v GC_INCR_GIANT=0 timeout 300 python profiles/incr_giant_probe.py > $out/${v}_g0_$r.json 2>&1
  done
done
