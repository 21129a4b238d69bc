#!/bin/bash
# What the giant filter costs in passed-through batches: bit probe (GC_GIANT_PT bit 0 off) vs marking (bit 1 off)
out=gpurun_out/r3d
mkdir -p $out
for r in 1 2; do
  for k in 0 1 2 3; do GC_GIANT_PT=$k timeout 300 python profiles/incr_giant_probe.py > $out/pt${k}_$r.json 2>&1; done
done
