#!/bin/bash
# usage (GPU box): bash tools/profile_box.sh TAG CONFIG [bench args]
# plain run, then the launch list and one ncu --set full capture of the timed kernel
tag=$1; cfg=$2; shift 2
cmd="python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline $*"
$cmd > gpurun_out/plain_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv $cmd > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ -s 3 -c 1 -o gpurun_out/prof_$tag $cmd > gpurun_out/ncu_$tag.log 2>&1
tail -2 gpurun_out/ncu_$tag.log
