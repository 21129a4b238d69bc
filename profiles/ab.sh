#!/bin/sh
# Quick A/B of bench.py variants (environment knobs) on one GPU.
run() {
  echo "== $1"
  env $1 python bench.py --skip-check --no-cpu-baseline --e2e-steps 0 --steps 60 --warmup 5 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.3e ms/step %.3f kout_ms %.3f launches/step %.1f' % (d['value'], d['ms_per_step'], r['kernel_ms'], d['launches_per_step']))"
}
for v in "$@"; do run "$v"; done
