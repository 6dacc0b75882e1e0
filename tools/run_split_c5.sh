#!/bin/bash
# GPU box: v6 per-role cycle split (DIAG instantiation) and skip-mode kernel times on a config
cfg=${1:-C5}; extra=${2:-}
for m in 0; do
  FEA_DEBUG_TIMING=1 FEA_DEBUG_MODE=$m timeout 300 python bench.py --config $cfg $extra --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dm.json 2>gpurun_out/dm.err
  python -c "
import json; d=json.load(open('gpurun_out/dm.json')); pc=d['config']['phase_cycles']; c=d['config']
nb=c['blocks']; print('DIAG mode $m', round(d['roofline']['kernel_ms_median'],3), 'blocks', nb)
for role in ('A_','B','P_'):
  tot=sum(v for k,v in pc.items() if k.startswith(role)) or 1
  print(role, ' '.join('%s=%.1f%%' % (k, 100.0*v/tot) for k,v in pc.items() if k.startswith(role) and v))
"
done
FEA_BUILD_DEFS="-DFEA6_DBGMODES" python -m paper_2204_03893_b200.build --force > /dev/null 2>&1 || exit 1
for m in ${MODES:-0 1 2 3 4 6 11}; do
  FEA_DEBUG_MODE=$m timeout 300 python bench.py --config $cfg $extra --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dm.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/dm.json')); print('skip mode $m', round(d['roofline']['kernel_ms_median'],3))"
done
