# v6 cost split (DIAG instantiation): kernel ms with parts skipped (FEA_DEBUG_MODE bits: 1 phase B,
# 2 A1, 4 A2, 8 producer gathers); results are wrong by design, timing only
for m in 0 1 2 4 8 3 5 6 7 15; do
  FEA_DEBUG_TIMING=1 FEA_DEBUG_MODE=$m python bench.py --config C5 --scale 1024 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dm.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/dm.json')); print('mode $m', round(d['roofline']['kernel_ms_median'],3))"
done
