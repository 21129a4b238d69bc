#!/bin/bash
out=gpurun_out/r3j
mkdir -p $out
timeout 300 python profiles/timeline.py forest_uniform27 1 > $out/tl_forest27.txt 2>&1
timeout 300 python profiles/timeline.py gridperm256:ldd+sv 1 > $out/tl_gridperm_ldd.txt 2>&1 || timeout 300 python profiles/timeline.py grid256:ldd+sv 1 > $out/tl_grid_ldd.txt 2>&1
