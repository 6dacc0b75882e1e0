#!/bin/bash
# GPU box: the C5 headline kernel -- plain bench run, ncu launch list (cold-cache, serialised), one
# ncu --set full capture of k_reassemble6 (each only after the previous command exited 0)
tag=${1:-r02_C5}; cfg=${2:-C5}
cmd="python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline"
$cmd > gpurun_out/${tag}_plain.json 2> gpurun_out/${tag}_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv $cmd > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_reassemble -s 3 -c 1 -o gpurun_out/${tag}_k $cmd > gpurun_out/${tag}_ncu.log 2>&1
echo rc=$?; tail -c 400 gpurun_out/${tag}_plain.json; tail -2 gpurun_out/${tag}_ncu.log
