#!/bin/bash
# GPU box, end of session 4: whole -m gpu suite, default bench line, per-config lines (matrix + tensor), two v6 block caps
tag=r02s4f
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${tag}_gputests.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/${tag}_bench.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for c in C2 C3 C4 C5 E2; do bash tools/bline.sh $c; done
for c in C2 C3 C4 C5; do bash tools/bline.sh $c --op tensor; done
bash tools/bline.sh C5 --tune 3=48
bash tools/bline.sh C3 --tune 3=96
timeout 300 python bench.py --config C4 --steps 20 --warmup 3 > gpurun_out/${tag}_bench_C4.json 2>/dev/null; tail -c 300 gpurun_out/${tag}_bench_C4.json
