#!/bin/bash
# GPU box, session 4: v5 L2 prefetch distance with the rounded blocks; k_tensor5 with 17 warps (e_max 1088)
bash tools/run_ab.sh "-DFEA5_PF=2;-DFEA5_PF=4;-DFEA5_PF=5" C4
FEA_BUILD_DEFS="-DFEA_T5_NW=17" python -m paper_2204_03893_b200.build --force > /dev/null 2>&1 || echo "build failed"
timeout 300 python -m pytest tests/test_gpu_tensor.py -x -q 2>&1 | tail -1
echo -n "T5_NW=17 "; bash tools/bline.sh C4 --op tensor
