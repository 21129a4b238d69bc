#!/bin/sh
# Quick A/B of bench.py variants (environment knobs) on one GPU.
#   sh profiles/ab.sh "" "GC_NO_SHORT_ROWS=1" "GC_L2_FETCH=32" ...
run() {
  echo "== $1"
  env $1 python bench.py --skip-check --no-cpu-baseline --e2e-steps 0 --steps 200 --warmup 5 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.3e ms/step %.4f kernel_ms %.4f launches/step %.1f clocks %s' % (d['value'], d['ms_per_step'], r['kernel_ms'], d['launches_per_step'], d['clocks']))"
}
for v in "$@"; do run "$v"; done
