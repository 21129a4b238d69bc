#!/bin/bash
out=gpurun_out
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 --timeout-method thread > $out/tests_r2e.log 2>&1
echo "tests rc=$?" >> $out/status_r2e.txt
GC_LDD_TRACE=1 timeout 300 python profiles/run_workload.py grid256:ldd+sv 1 > $out/ldd_trace.log 2>&1
GC_LDD_TRACE=1 timeout 300 python profiles/run_workload.py gridperm256:ldd+sv 1 >> $out/ldd_trace.log 2>&1
timeout 600 python bench_configs.py --configs 3 --cpu 0 --reps 3 \
    --specs ldd+sv,none+sv,ldd\(0.5\)+sv --out $out/ldd_r2e.jsonl > $out/ldd_r2e.log 2>&1
echo "ldd rc=$?" >> $out/status_r2e.txt
