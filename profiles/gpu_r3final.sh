#!/bin/bash
# Final check of HEAD on a fresh box: GPU suite, smoke, headline bench.
out=gpurun_out/r3final
mkdir -p $out
st=$out/status.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 --timeout-method thread > $out/tests.txt 2>&1; echo "tests rc=$?" >> $st
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1; echo "smoke rc=$?" >> $st
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" >> $st
