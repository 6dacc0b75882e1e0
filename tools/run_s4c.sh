#!/bin/bash
# GPU box, session 4: P1 warp count with blocks rounded to whole unit rounds
bash tools/run_ab.sh "-DFEA5_NW1=21;-DFEA5_NW1=22;-DFEA5_NW1=23;-DFEA5_NW1=16;-DFEA5_NW1=18" C4
