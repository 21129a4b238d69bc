#!/bin/bash
# Round-2 closing evidence refresh after the re-entry changes (tag r3z): tests, smoke, headline bench + reference
# arm, every BASELINE config with same-run CPU baselines, launch list, ncu of
# the headline and incremental kernels, shard models, single-GPU scale sweep.
out=gpurun_out/r3z
mkdir -p $out
st=$out/status.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 --timeout-method thread > $out/tests.txt 2>&1; echo "tests rc=$?" >> $st
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1; echo "smoke rc=$?" >> $st
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" >> $st
timeout 900 python bench.py --impl reference > $out/bench_reference.json 2> $out/bench_reference.err; echo "ref rc=$?" >> $st
timeout 2400 python bench_configs.py --out $out/configs.jsonl > $out/configs.log 2>&1; echo "configs rc=$?" >> $st
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 3 --warmup 3 --skip-check --no-cpu-baseline --e2e-steps 0 > $out/launches_bench.log 2>&1; echo "launches rc=$?" >> $st
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_union_rows -s 4 -c 1 \
  -o $out/prof_kout -f python profiles/run_workload.py kout_s24 3 > $out/prof_kout.log 2>&1; echo "ncu kout rc=$?" >> $st
GC_INCR_GIANT=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_giant_compact|k_union_coo_async_mlp" -s 90 -c 2 \
  -o $out/prof_incr -f python profiles/incr_giant_probe.py > $out/prof_incr.log 2>&1; echo "ncu incr rc=$?" >> $st
timeout 900 python profiles/single_scale.py 24 25 26 27 > $out/single_scale.jsonl 2>&1; echo "single rc=$?" >> $st
timeout 1200 python profiles/shard_model.py --ranks 1,2,4,8 --check > $out/shard_model.jsonl 2> $out/shard_model.err; echo "shard rc=$?" >> $st
timeout 1200 python profiles/shard_model.py --incremental --ranks 1,2,4,8 --check > $out/shard_model_incremental.jsonl 2> $out/shard_model_incremental.err; echo "shard incr rc=$?" >> $st
for g in 1 0; do GC_INCR_GIANT=$g timeout 300 python profiles/incr_giant_probe.py > $out/incr_giant$g.json 2>&1; done; echo "giant rc=$?" >> $st
for t in memcheck racecheck; do timeout 1200 compute-sanitizer --tool $t --print-limit 20 python profiles/sanitize_workload.py > $out/$t.txt 2>&1; echo "$t rc=$?" >> $st; done
timeout 1200 python profiles/shard_model.py --bfs --ranks 1,2,4,8 --check > $out/shard_model_bfs_forest.jsonl 2> $out/shard_model_bfs.err; echo "shard bfs rc=$?" >> $st
