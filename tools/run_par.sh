#!/bin/bash
# GPU box: parity suite with failure details, then quick numbers for the given configs
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --tb=short 2>&1 | tail -30
for c in "$@"; do bash tools/bline.sh $c; done
