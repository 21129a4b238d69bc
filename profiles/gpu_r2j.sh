#!/bin/bash
out=gpurun_out
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 --timeout-method thread > $out/tests_r2j.log 2>&1
echo "tests rc=$?" >> $out/status_r2j.txt
for v in 1 0; do
  GC_BFS_PERSIST=$v timeout 900 python bench_configs.py --configs 3,5 --cpu 0 --reps 3 \
    --specs bfs+sv,bfs+async+halve,ldd+sv --out $out/bfsj_persist$v.jsonl > $out/bfsj_persist$v.log 2>&1
  echo "bfs$v rc=$?" >> $out/status_r2j.txt
done
