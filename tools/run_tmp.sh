python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
FEA_DEBUG_TIMING=1 python bench.py --config C5 --scale 1024 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/diag_c5s1024d.json
python -c "
import json; d=json.load(open('gpurun_out/diag_c5s1024d.json')); print(d['config']['phase_cycles'])"
for a in "--config C5 --scale 1024" "--config C5" "--config C3"; do python bench.py $a --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/t.json 2>gpurun_out/t.err; python -c "
import json; d=json.load(open('gpurun_out/t.json')); print(d['config']['workload'][:40], d['roofline']['kernel_ms_median'], d['roofline']['frac'], d['config']['elem_visits_over_owned'])"; done
