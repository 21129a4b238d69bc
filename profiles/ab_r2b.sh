#!/bin/bash
# r2b: GPU suite (per-test timeout) + A/B of the round-2 kernel changes
out=gpurun_out
mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 300 --timeout-method thread > $out/tests_r2b.log 2>&1
echo "tests rc=$?" >> $out/status_r2b.txt
for v in 0 1; do
  GC_LDD_PERSIST=$v timeout 600 python bench_configs.py --configs 3 --cpu 0 --reps 3 \
    --specs ldd+sv,ldd+lt_prs,none+sv,ldd\(0.5\)+sv --out $out/ldd_persist$v.jsonl > $out/ldd_persist$v.log 2>&1
  echo "ldd$v rc=$?" >> $out/status_r2b.txt
done
for k in 0 2 4 8; do
  GC_COO_MLP=$k timeout 600 python bench_configs.py --configs 4 --cpu 0 --reps-incr 2 \
    --specs none+async+halve --out $out/mlp$k.jsonl > $out/mlp$k.log 2>&1
  echo "mlp$k rc=$?" >> $out/status_r2b.txt
done
sh profiles/ab.sh "" "GC_P_EVICT_LAST=1" "" "GC_P_EVICT_LAST=1" > $out/ab_evict.txt 2>&1
