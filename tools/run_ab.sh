#!/bin/bash
# GPU box A/B: bash tools/run_ab.sh "<defs B>;<defs C>;..." [configs...] -- the in-tree build (A),
# then one rebuild per ;-separated FEA_BUILD_DEFS variant; tools/bline.sh per config for each
IFS=';' read -ra vars <<< "$1"; shift; cfgs="${@:-C5 C3}"
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for c in $cfgs; do echo -n "A "; bash tools/bline.sh $c; done
for defs in "${vars[@]}"; do
  FEA_BUILD_DEFS="$defs" python -m paper_2204_03893_b200.build --force > /dev/null 2>&1 || { echo "build $defs failed"; continue; }
  echo -n "B($defs) parity: "; timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
  for c in $cfgs; do echo -n "B($defs) "; bash tools/bline.sh $c; done
done
