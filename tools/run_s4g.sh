#!/bin/bash
# GPU box, session 4: P2 block caps (whole rounds of units), then P4 with the split A1 (A1MODE 4)
bash tools/bline.sh C2 --tune 3=256
bash tools/bline.sh C2 --tune 3=224
bash tools/bline.sh E2 --tune 3=256
bash tools/run_ab.sh "-DFEA6_A1MODE_P4=4;-DFEA6_A1MODE_P4=4 -DFEA6_A1A=2;-DFEA6_A1MODE_P4=4 -DFEA6_A1A=1" C5
