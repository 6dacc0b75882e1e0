#!/bin/bash
# GPU box, session 4: e_max rounded to whole rounds of 32-element units over the warps (P1 kernels);
# explicit FEA_TUNE_EMAX values are taken as given (3=1520 / 3=1144 = the previous defaults)
bash tools/bline.sh C4
bash tools/bline.sh C4 --tune 3=1520
bash tools/bline.sh C4 --tune 3=1272
bash tools/bline.sh C4 --op tensor
bash tools/bline.sh C4 --op tensor --tune 3=1144
bash tools/bline.sh C4 --op tensor --tune 3=512
timeout 900 python -m pytest tests -m gpu -x -q -k "C4 or p1 or P1 or tensor or small or determin" > gpurun_out/s4b_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s4b_tests.log
