#!/bin/sh
# Quick A/B of bench.py variants (environment knobs) on one GPU.
#   sh profiles/ab.sh "" "GC_SOME_KNOB=1" ...
run() {
  echo "== $1"
  env $1 python bench.py --skip-check --no-cpu-baseline --e2e-steps 0 --steps 200 --warmup 5 > /tmp/ab.out 2> /tmp/ab.err
  rc=$?
  tail -1 /tmp/ab.out | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.3e ms/step %.4f kernel_ms %.4f launches/step %.1f clocks %s' % (d['value'], d['ms_per_step'], r['kernel_ms'], d['launches_per_step'], d['clocks']))" || { echo "rc=$rc"; tail -5 /tmp/ab.err; }
}
for v in "$@"; do run "$v"; done
