timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "config_parity_small or single_and_two or distinct or more_than" 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -12
FEA_DEBUG_TIMING=1 python bench.py --config C5 --scale 1024 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/diag_c5s1024d.json
python -c "
import json; d=json.load(open('gpurun_out/diag_c5s1024d.json')); pc=d['config']['phase_cycles']
A=sum(v for k,v in pc.items() if k.startswith('A_')); B=sum(v for k,v in pc.items() if k.startswith('B'))
print({k: round(100*v/A,1) for k,v in pc.items() if k.startswith('A_')}); print({k: round(100*v/B,1) for k,v in pc.items() if k.startswith('B')}); print(d['roofline']['kernel_ms_median'])"
