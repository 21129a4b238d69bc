#!/bin/bash
out=gpurun_out/r3e
mkdir -p $out
GC_GIANT_PT=1 timeout 300 python profiles/timeline.py incrp26:none+async+halve:10 1 > $out/tl_pt1.txt 2>&1
GC_INCR_GIANT=0 timeout 300 python profiles/timeline.py incrp26:none+async+halve:10 1 > $out/tl_g0.txt 2>&1
