#!/bin/bash
out=gpurun_out
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 --timeout-method thread > $out/tests_r2g.log 2>&1
echo "tests rc=$?" >> $out/status_r2g.txt
sh profiles/ab.sh "" "GC_MODE_COOP=0" "" "GC_MODE_COOP=0" > $out/ab_r2g.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_union_rows -s 0 -c 1 \
    -o $out/prof_kout -f python profiles/run_workload.py kout_s24 1 > $out/prof_kout.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_post_sample|k_mode_fallback" -s 0 -c 2 \
    -o $out/prof_post2 -f python profiles/run_workload.py kout_s24 1 > $out/prof_post2.log 2>&1
echo "prof rc=$?" >> $out/status_r2g.txt
