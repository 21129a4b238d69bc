#!/bin/bash
# One gpurun call: GPU tests, headline bench, per-config bench, ncu launch list
# and one full ncu capture of the dominant kernel.  Outputs in gpurun_out/.
#   gpurun --timeout 2400 -- 'bash profiles/gpu_round.sh [tag] [parts]'
# parts: comma list of tests,bench,configs,launches,full (default: all)
tag=${1:-r1}
parts=${2:-tests,bench,configs,launches,full}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $out/gpu_$tag.txt 2>&1
has() { case ",$parts," in *",$1,"*) return 0;; esac; return 1; }
if has tests; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $out/tests_$tag.log 2>&1; echo "tests rc=$?" >> $out/status_$tag.txt
fi
if has bench; then
  timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench rc=$?" >> $out/status_$tag.txt
fi
if has configs; then
  rm -f $out/configs_$tag.jsonl
  timeout 1500 python bench_configs.py --out $out/configs_$tag.jsonl > $out/configs_$tag.log 2>&1; echo "configs rc=$?" >> $out/status_$tag.txt
fi
if has launches; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_$tag.csv \
    python bench.py --steps 3 --warmup 3 --skip-check --no-cpu-baseline --e2e-steps 0 > $out/launches_bench_$tag.log 2>&1
  echo "launches rc=$?" >> $out/status_$tag.txt
fi
if has full; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_union_rows -s 4 -c 2 \
    -o $out/prof_kout_$tag -f python profiles/run_workload.py kout_s24 3 > $out/prof_kout_$tag.log 2>&1
  echo "full rc=$?" >> $out/status_$tag.txt
fi
