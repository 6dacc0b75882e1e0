for m in 0 3 7; do
  FEA_DEBUG_TIMING=1 FEA_DEBUG_MODE=$m python bench.py --config C5 --scale 1024 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dm.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/dm.json')); pc=d['config']['phase_cycles']
A=sum(v for k,v in pc.items() if k.startswith('A_')); B=sum(v for k,v in pc.items() if k.startswith('B')); P=pc['P_free_wait']+pc['P_gather']
n=8*148*14*580
print('mode $m', round(d['roofline']['kernel_ms_median'],3), 'A per-warp-block cycles', {k: round(v/n) for k,v in pc.items() if k.startswith('A_') and v}, 'P', round(pc['P_free_wait']/(n/8)), round(pc['P_gather']/(n/8)))"
done
