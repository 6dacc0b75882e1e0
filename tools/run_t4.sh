#!/bin/bash
# GPU box: tensor tests, then the tensor timings per config
tag=${1:-t4}
timeout 900 python -m pytest tests/test_gpu_tensor.py -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tensor tests rc=$?"; tail -2 gpurun_out/${tag}_tests.log
for c in ${CFGS:-C2 C3 C5}; do bash tools/bline.sh $c --op tensor; done
