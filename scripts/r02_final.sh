#!/bin/bash
# Final validation pass of the round (under gpurun from the repo root): GPU suite, smoke,
# default bench line.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${TAG:-r02f}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.txt 2>&1; echo "gpu tests rc=$?"; tail -2 $O/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.txt
timeout 600 python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('$O/bench_cfg4.json'));print(round(d['value'],1),round(d['e2e']['value'],1),d['clocks'],round(d['roofline']['frac'],3))"
