#!/bin/bash
# GPU box, session 4: bounds-check build (tools/sanitize.sh) plus the full-size C4 tests (the P1
# blocks in whole unit rounds: e_max 1280 / 1024) under the same build
bash tools/sanitize.sh
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "C4" > gpurun_out/chk_fullC4.log 2>&1; echo "== fullsize C4 rc=$?"; tail -3 gpurun_out/chk_fullC4.log
grep -c "FEA_CHECK failed" gpurun_out/chk_fullC4.log
