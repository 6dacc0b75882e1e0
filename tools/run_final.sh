#!/bin/bash
# GPU box, end of round: whole -m gpu suite, the default bench line, per-config numbers, the C5
# launch list and one ncu --set full capture of k_reassemble6 (each after its command exited 0)
tag=${1:-r02f}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${tag}_gputests.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"; tail -c 700 gpurun_out/${tag}_bench.json
for c in C2 C3 C4 C5 E2; do bash tools/bline.sh $c; done
cmd="python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_C5_launches.csv $cmd > /dev/null 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_reassemble6 -s 3 -c 1 -o gpurun_out/${tag}_C5_k $cmd > gpurun_out/${tag}_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/${tag}_ncu.log
