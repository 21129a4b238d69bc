#!/bin/bash
out=gpurun_out
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 --timeout-method thread > $out/tests_r2h.log 2>&1
echo "tests rc=$?" >> $out/status_r2h.txt
sh profiles/ab.sh "" "" > $out/ab_r2h.txt 2>&1
for v in 1 0; do
  GC_BFS_PERSIST=$v timeout 900 python bench_configs.py --configs 3,5 --cpu 0 --reps 3 \
    --specs bfs+sv,bfs+async+halve,none+sv --no-permuted --out $out/bfs_persist$v.jsonl > $out/bfs_persist$v.log 2>&1
  echo "bfs$v rc=$?" >> $out/status_r2h.txt
done
