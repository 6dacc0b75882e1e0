#!/bin/bash
# usage: tools/sweep.sh CONFIG "tune-args-1" "tune-args-2" ...   (run on the GPU box)
cfg=$1; shift
for t in "$@"; do
  args=""; for kv in $t; do args="$args --tune $kv"; done
  timeout 300 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline $args > /tmp/sw.json 2>/tmp/sw.err
  python -c "import json; d=json.load(open('/tmp/sw.json')); c=d['config']; print('$cfg', '[$t]', 'ms=%.4f frac=%.3f blocks=%d visits=%.3f smem=%d grid=%d' % (d['ms_per_step'], d['roofline']['frac'], c['blocks'], c['elem_visits_over_owned'], c['smem_per_cta'], c['grid']))" || tail -3 /tmp/sw.err
done
