#!/bin/bash
# GPU box: compute-sanitizer is closed on this pool, so every kernel runs in the FEA_BOUNDS_CHECK build
# (device-side checks of the shared- and global-memory indices, fea_device.cuh FEA_CHECK) on the small
# cases of tools/sanitize_cases.py (each also checked against the oracle) and the -m gpu parity tests.
FEA_BUILD_DEFS="-DFEA_BOUNDS_CHECK" python -m paper_2204_03893_b200.build --force > gpurun_out/chk_build.log 2>&1 || { tail gpurun_out/chk_build.log; exit 1; }
python tools/sanitize_cases.py > gpurun_out/chk_cases.log 2>&1; echo "== cases rc=$?"; tail -3 gpurun_out/chk_cases.log
python -m pytest tests/test_gpu_parity.py tests/test_gpu_tensor.py tests/test_dist_gpu.py -q -x > gpurun_out/chk_tests.log 2>&1; echo "== tests rc=$?"; tail -3 gpurun_out/chk_tests.log
grep -c "FEA_CHECK failed" gpurun_out/chk_cases.log gpurun_out/chk_tests.log
