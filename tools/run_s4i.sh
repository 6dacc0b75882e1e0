#!/bin/bash
# GPU box, session 4: P1 M+K (the C1 recipe on a 2048 x 2048 grid): rounded blocks (e_max 640) vs the
# previous default (928); diagnostics only (--scale), not a bench value
bash tools/bline.sh C1 --scale 2048
bash tools/bline.sh C1 --scale 2048 --tune 3=928
bash tools/bline.sh C1 --scale 2048 --tune 3=800
