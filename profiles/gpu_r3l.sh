#!/bin/bash
out=gpurun_out/r3l
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 --timeout-method thread > $out/tests.txt 2>&1; echo "tests rc=$?" >> $out/status.txt
