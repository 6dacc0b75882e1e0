#!/bin/bash
# GPU box: k_tensor5 tests, C4 tensor timing (default build), then other warp counts (rebuilds)
tag=${1:-t5c}
timeout 900 python -m pytest tests/test_gpu_tensor.py -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tensor tests rc=$?"; tail -2 gpurun_out/${tag}_tests.log
bash tools/bline.sh C4 --op tensor; bash tools/bline.sh C2 --op tensor --tune 8=4
for nw in ${NWS:-16}; do
  FEA_BUILD_DEFS="-DFEA_T5_NW=$nw $DEFS" python -m paper_2204_03893_b200.build --force > gpurun_out/${tag}_build$nw.log 2>&1 && bash tools/bline.sh C4 --op tensor && echo "(NW=$nw)"
done
