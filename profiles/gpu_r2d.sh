#!/bin/bash
out=gpurun_out
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 400 --timeout-method thread > $out/tests_r2d.log 2>&1
echo "tests rc=$?" >> $out/status_r2d.txt
timeout 600 python bench_configs.py --configs 3 --cpu 0 --reps 3 \
    --specs ldd+sv,ldd+lt_prs,none+sv,ldd\(0.5\)+sv,ldd\(0.1\)+sv --out $out/ldd_r2d.jsonl > $out/ldd_r2d.log 2>&1
echo "ldd rc=$?" >> $out/status_r2d.txt
sh profiles/ab.sh "" > $out/ab_r2d.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ldd_persist -c 1 \
  -o $out/prof_ldd_perm -f python profiles/run_workload.py gridperm256:ldd+sv 1 > $out/prof_ldd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ldd_persist -c 1 \
  -o $out/prof_ldd_nat -f python profiles/run_workload.py grid256:ldd+sv 1 >> $out/prof_ldd.log 2>&1
echo "prof rc=$?" >> $out/status_r2d.txt
