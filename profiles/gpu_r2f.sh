#!/bin/bash
# r2f: every BASELINE config with its same-run CPU baseline, the bench launch
# list, and one ncu --set full capture per hot kernel
out=gpurun_out
mkdir -p $out
rm -f $out/configs_r2f.jsonl
timeout 2400 python bench_configs.py --out $out/configs_r2f.jsonl > $out/configs_r2f.log 2>&1
echo "configs rc=$?" >> $out/status_r2f.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_r2f.csv \
  python bench.py --steps 3 --warmup 3 --skip-check --no-cpu-baseline --e2e-steps 0 > $out/launches_bench_r2f.log 2>&1
echo "launches rc=$?" >> $out/status_r2f.txt
cap() {  # name kernel-regex skip count workload
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c $4 \
    -o $out/prof_$1 -f python profiles/run_workload.py $5 1 > $out/prof_$1.log 2>&1
  echo "prof $1 rc=$?" >> $out/status_r2f.txt
}
cap kout k_union_rows 2 1 kout_s24
cap incr k_union_coo 20 1 incr_s26
cap ldd k_ldd_persist 0 1 grid256:ldd+sv
cap bfsbu k_bfs_bu 0 2 bfs_uniform27
cap bfstd "k_bfs_td" 0 3 bfs_uniform27
cap sv k_sv_hook 0 3 gridperm256:none+sv
cap post k_post_sample 0 1 kout_s24
