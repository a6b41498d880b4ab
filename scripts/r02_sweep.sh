#!/bin/bash
# BASELINE configs[4] throughput / occupancy sweep on one box (under gpurun from the repo root):
# foreground 5/25/60/95 % x stride 512/384/256 and, at 95 % / stride 256, batch 64-512 windows
# per launch; the batch-invariance GPU test first (the batch sizes the sweep times are checked
# bit-identical against batch 64, which test_gpu_fullsize checks against the oracle).
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${TAG:-r02s}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_batch.py -q -s > $O/gpu_batch_test.txt 2>&1; echo "batch test rc=$?"
tail -3 $O/gpu_batch_test.txt
for fg in 5 25 60 95; do
  for s in 512 384 ""; do
    wl=cfg5_fg$fg${s:+_s$s}
    timeout 600 python bench.py --workload $wl --no-cpu --steps 2 > $O/bench_$wl.json 2> $O/bench_$wl.err
    echo "$wl rc=$? $(python -c "import json;d=json.load(open('$O/bench_$wl.json'));print(d['config']['kept_tiles'],round(d['value'],1),round(d['e2e']['value'],1),d['clocks']['sm_mhz'])" 2>&1)"
  done
done
for b in 64 128 256 512; do
  wl=cfg5_fg95
  timeout 600 python bench.py --workload $wl --batch $b --no-cpu --steps 2 > $O/bench_${wl}_b$b.json 2> $O/bench_${wl}_b$b.err
  echo "$wl b$b rc=$? $(python -c "import json;d=json.load(open('$O/bench_${wl}_b$b.json'));print(d['config']['kept_tiles'],round(d['value'],1),round(d['e2e']['value'],1),d['clocks']['sm_mhz'])" 2>&1)"
done
