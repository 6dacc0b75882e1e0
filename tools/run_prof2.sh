#!/bin/bash
# GPU box: ncu --set full of k_reassemble6 on C5@1024, production build and the pure-A2 skip mode (11)
bash tools/prof_cfg.sh c5s_prod "--config C5 --scale 1024" regex:k_reassemble6
FEA_BUILD_DEFS="-DFEA6_DBGMODES" python -m paper_2204_03893_b200.build --force > /dev/null 2>&1 || exit 1
FEA_DEBUG_MODE=11 bash tools/prof_cfg.sh c5s_m11 "--config C5 --scale 1024" regex:k_reassemble6
