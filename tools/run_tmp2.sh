timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "config_parity_small or single_and_two or distinct or more_than" 2>&1 | tail -3
bash tools/run_tmp.sh
