#!/bin/bash
# usage (GPU box): bash tools/bline.sh CONFIG [bench args]  -- one summary line per run
c=$1; shift
timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline "$@" 2>/tmp/b.err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']
print('$c', '$*', 'ms=%.4f frac=%.3f blocks=%d visits=%.3f smem=%d grid=%d kern=%s l2=%s' % (d['ms_per_step'], d['roofline']['frac'], c['blocks'], c['elem_visits_over_owned'], c['smem_per_cta'], c['grid'], d['roofline']['kernel'], c['l2'][:12]))" || tail -3 /tmp/b.err
