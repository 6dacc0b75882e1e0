#!/bin/bash
# GPU box, session 4: zero-code experiments (one-matrix plans = two passes with larger blocks; v5 block caps)
bash tools/bline.sh C5 --tune 4=1
bash tools/bline.sh C5 --tune 4=2
bash tools/bline.sh C3 --tune 4=1
bash tools/bline.sh C3 --tune 4=2
for e in 640 960 1280 1920; do bash tools/bline.sh C4 --tune 3=$e; done
bash tools/bline.sh C4 --tune 1=110000
bash tools/bline.sh C4 --tune 1=150000
bash tools/bline.sh C2 --tune 1=110000
