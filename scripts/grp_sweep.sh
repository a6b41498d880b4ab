#!/bin/bash
# Grouped-schedule sweep on the GPU box (under gpurun from the repo root).
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${TAG:-s2}; mkdir -p $O
python -m pytest tests/test_gpu_grouped.py -x -q -s > $O/grouped_tests.txt 2>&1; echo "grouped tests rc=$?"
for g in ${GRPS:-0 1 2 4}; do
  for gl in ${GLEVS:-2}; do
    timeout 300 python scripts/layer_profile.py cfg4 fp16f8 2 grp=$g glev=$gl > $O/layers_g${g}_l${gl}.txt 2>&1; echo "layers grp=$g glev=$gl rc=$? $(head -1 $O/layers_g${g}_l${gl}.txt)"
  done
done
for g in ${BENCH_GRPS:-1}; do
  python bench.py --no-cpu --arch grp=$g > $O/bench_g$g.json 2> $O/bench_g$g.err; echo "bench grp=$g rc=$? $(tail -c 400 $O/bench_g$g.json | head -c 200)"
done
