#!/bin/bash
# BFS frontier-expansion kernels: min resident blocks 1 (40 registers) / 7 / 8 (32 registers, spills)
out=gpurun_out/r3g
mkdir -p $out
for r in 1 2; do
  for v in t1 t7 t8; do
    GC_LIB_VARIANT=$v timeout 300 python profiles/bfs_time.py 27 bfs+async+halve > $out/${v}_c5_$r.txt 2>&1
  done
done
for v in t1 t8; do GC_LIB_VARIANT=$v timeout 300 python profiles/timeline.py grid256:bfs+sv 1 | tail -1 > $out/${v}_grid.txt 2>&1; done
