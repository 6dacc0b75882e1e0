# quick perf check: C5@1024 diagnostic, C5, C3 (kernel ms, frac, visits)
for a in "--config C5 --scale 1024" "--config C5" "--config C3"; do python bench.py $a --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/t.json 2>gpurun_out/t.err; python -c "
import json; d=json.load(open('gpurun_out/t.json')); print(d['config']['workload'][:40], d['roofline']['kernel_ms_median'], d['roofline']['frac'], d['config']['elem_visits_over_owned'])"; done
