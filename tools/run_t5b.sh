#!/bin/bash
# GPU box: k_tensor5 ncu capture on C4 (default build), then the warp-count sweep (rebuilds)
tag=${1:-t5b}
cmd="python bench.py --config C4 --op tensor --steps 3 --warmup 3 --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:k_tensor5 -s 3 -c 1 -o gpurun_out/${tag}_C4_k_tensor5 $cmd > gpurun_out/${tag}_ncu.log 2>&1; echo "ncu rc=$?"; tail -1 gpurun_out/${tag}_ncu.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_C4_tensor_launches.csv $cmd > /dev/null 2>&1; echo "launches rc=$?"
for nw in 12 20; do
  FEA_BUILD_DEFS="-DFEA_T5_NW=$nw" python -m paper_2204_03893_b200.build --force > gpurun_out/${tag}_build$nw.log 2>&1 && bash tools/bline.sh C4 --op tensor --tune 8=5 && echo "(NW=$nw)"
done
