#!/bin/bash
# Re-entry check of HEAD: GPU tests, smoke, headline bench, reference arm.
out=gpurun_out
mkdir -p $out
tag=${1:-r2k}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $out/gpu_$tag.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 --timeout-method thread > $out/tests_$tag.log 2>&1
echo "tests rc=$?" >> $out/status_$tag.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_$tag.log 2>&1
echo "smoke rc=$?" >> $out/status_$tag.txt
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err
echo "bench rc=$?" >> $out/status_$tag.txt
timeout 900 python bench.py --impl reference > $out/bench_ref_$tag.json 2> $out/bench_ref_$tag.err
echo "ref rc=$?" >> $out/status_$tag.txt
