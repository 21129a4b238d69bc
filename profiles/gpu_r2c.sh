#!/bin/bash
out=gpurun_out
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 400 --timeout-method thread > $out/tests_r2c.log 2>&1
echo "tests rc=$?" >> $out/status_r2c.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_incr26.csv \
  python profiles/run_workload.py incr_s26 1 > $out/launches_incr26.log 2>&1
echo "launches rc=$?" >> $out/status_r2c.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ldd_persist -c 1 \
  -o $out/prof_ldd_persist -f python profiles/run_workload.py gridperm256:ldd+sv 1 > $out/prof_ldd.log 2>&1
echo "ldd prof rc=$?" >> $out/status_r2c.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_union_coo -s 10 -c 1 \
  -o $out/prof_incr -f python profiles/run_workload.py incr_s26 1 > $out/prof_incr.log 2>&1
echo "incr prof rc=$?" >> $out/status_r2c.txt
sh profiles/ab.sh "" "GC_P_EVICT_LAST=1" "" "GC_P_EVICT_LAST=1" > $out/ab_evict.txt 2>&1
