#!/bin/bash
# A/B of the giant-filter bitmap's L2 evict_last hint (GC_GIANT_KEEP) on the config-4 stream
out=gpurun_out/r3b
mkdir -p $out
for r in 1 2; do
  for k in 1 0; do GC_GIANT_KEEP=$k timeout 300 python profiles/incr_giant_probe.py > $out/keep${k}_$r.json 2>&1; done
done
GC_GIANT_KEEP=1 timeout 300 python profiles/incr_giant_probe.py none+rem_cas+halve+split > $out/remcas_keep1.json 2>&1
GC_GIANT_KEEP=0 timeout 300 python profiles/incr_giant_probe.py none+rem_cas+halve+split > $out/remcas_keep0.json 2>&1
timeout 600 python -m pytest tests/test_gpu_incremental.py tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider > $out/tests.txt 2>&1; echo "tests rc=$?" >> $out/status.txt
