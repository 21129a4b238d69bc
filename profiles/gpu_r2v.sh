#!/bin/bash
# compute-sanitizer on the round-2 kernels (giant filter, merge flags,
# list finalize, list root snapshot) via the sanitizer workload
out=gpurun_out/r2v
mkdir -p $out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python profiles/sanitize_workload.py > $out/$tool.txt 2>&1
  echo "$tool rc=$?" >> $out/status.txt
done
