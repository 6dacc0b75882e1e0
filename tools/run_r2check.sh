#!/bin/bash
# GPU box: full -m gpu suite, the default bench line, per-config quick numbers
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_gputests.log
timeout 400 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/r2_bench_default.json
for c in C2 C3 C4 C5 E2; do bash tools/bline.sh $c; done
for c in C2 C3 C4 C5; do bash tools/bline.sh $c --op tensor; done
