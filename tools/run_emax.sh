#!/bin/bash
# GPU box: element cap per row block (FEA_TUNE_EMAX = 3) on the small configs (few blocks per SM)
for c in E2 C1; do bash tools/bline.sh $c; for e in 48 96 160 256; do bash tools/bline.sh $c --tune 3=$e; done; done
bash tools/bline.sh C2; for e in 200 300 450; do bash tools/bline.sh C2 --tune 3=$e; done
bash tools/bline.sh E2 --op tensor; for e in 48 96; do bash tools/bline.sh E2 --op tensor --tune 3=$e; done
