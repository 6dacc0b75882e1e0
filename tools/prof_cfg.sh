#!/bin/bash
# usage (GPU box): bash tools/prof_cfg.sh TAG "bench args" [kernel-regex]
# plain run, then one ncu --set full capture of the timed kernel (the plain run must exit 0 first)
tag=$1; args=$2; kre=${3:-regex:k_}
cmd="python bench.py --steps 3 --warmup 3 --no-cpu-baseline $args"
$cmd > gpurun_out/plain_$tag.json 2> gpurun_out/plain_$tag.err && \
ncu --set full --clock-control none --import-source on -k $kre -s 3 -c 1 -o gpurun_out/prof_$tag $cmd > gpurun_out/ncu_$tag.log 2>&1
tail -c 600 gpurun_out/plain_$tag.json; tail -2 gpurun_out/ncu_$tag.log
