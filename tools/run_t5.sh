#!/bin/bash
# GPU box: k_tensor5 parity (tensor tests, full-size C4 tensor window) and C4 tensor timings vs k_tensor
tag=${1:-t5}
timeout 900 python -m pytest tests/test_gpu_tensor.py -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tensor tests rc=$?"; tail -2 gpurun_out/${tag}_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "tensor and C4" > gpurun_out/${tag}_full.log 2>&1; echo "fullsize rc=$?"; tail -2 gpurun_out/${tag}_full.log
for t in 5 1; do bash tools/bline.sh C4 --op tensor --tune 8=$t; done
for nw in 12 20; do
  FEA_BUILD_DEFS="-DFEA_T5_NW=$nw" python -m paper_2204_03893_b200.build --force > /dev/null 2>&1 && bash tools/bline.sh C4 --op tensor --tune 8=5 && echo "(NW=$nw)"
done
