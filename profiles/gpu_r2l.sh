#!/bin/bash
# Incremental giant filter: tests + config 4 with the filter on / off.
out=gpurun_out
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "incr or config or distributed or comm" --timeout 400 > $out/tests_r2l.log 2>&1
echo "tests rc=$?" >> $out/status_r2l.txt
for g in 1 0; do
  GC_INCR_GIANT=$g timeout 900 python bench_configs.py --configs 4 --cpu 0 --specs none+async+halve,none+rem_cas+halve+split \
    --out $out/incr_giant$g.jsonl > $out/incr_giant$g.log 2>&1
  echo "giant$g rc=$?" >> $out/status_r2l.txt
done
