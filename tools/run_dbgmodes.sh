# production instantiation with the skip bits compiled in (-DFEA6_DBGMODES): kernel ms per skip mode
FEA_BUILD_DEFS="-DFEA6_DBGMODES" python -m paper_2204_03893_b200.build --force > /dev/null 2>&1 || exit 1
for m in ${MODES:-0 1 2 4 8 3 5 6 9 10 12}; do
  FEA_DEBUG_MODE=$m python bench.py --config C5 --scale 1024 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dm.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/dm.json')); print('mode $m', round(d['roofline']['kernel_ms_median'],3))"
done
