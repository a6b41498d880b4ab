#!/bin/bash
# Round-2 measurement pass on the GPU box (run under gpurun from the repo root).
# Every ncu command follows a plain run of the same command that exited 0.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
TAG=${TAG:-r02c}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python bench.py > gpurun_out/${TAG}_bench_cfg4.json 2> gpurun_out/${TAG}_bench_cfg4.err; echo "bench rc=$?"
python bench.py --profile-only --no-cpu --no-e2e > gpurun_out/${TAG}_prof.json 2>&1; echo "profile-only rc=$?"
$NCU --metrics $M --clock-control none --kernel-name-base demangled -k regex:"conv|stem" --launch-skip 200 \
  --launch-count 290 --csv --log-file gpurun_out/${TAG}_cfg4_conv.csv \
  python bench.py --profile-only --no-cpu --no-e2e > gpurun_out/${TAG}_ncu1.log 2>&1; echo "ncu conv rc=$?"
$NCU --metrics $M --clock-control none --kernel-name-base demangled \
  -k regex:"pyramid|median|hist_kernel|otsu|fg_kernel|tile_keep|compact|finalize|pad_colour|gap_kernel|controller" \
  --launch-count 420 --csv --log-file gpurun_out/${TAG}_cfg4_front.csv \
  python bench.py --profile-only --no-cpu --no-e2e > gpurun_out/${TAG}_ncu2.log 2>&1; echo "ncu front rc=$?"
$NCU --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"conv3_nz_kernel<__half, \\(int\\)32, \\(int\\)8, \\(int\\)2, \\(int\\)4" --launch-skip 3 -c 1 -o /tmp/${TAG}_head -f \
  python bench.py --profile-only --no-cpu --no-e2e > gpurun_out/${TAG}_ncu3.log 2>&1; echo "ncu head rc=$?"
$NCU -i /tmp/${TAG}_head.ncu-rep --page raw --csv > gpurun_out/${TAG}_head_raw.csv 2>/dev/null
$NCU --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"stem_tc" --launch-skip 3 -c 1 -o /tmp/${TAG}_stem -f \
  python bench.py --profile-only --no-cpu --no-e2e > gpurun_out/${TAG}_ncu4.log 2>&1; echo "ncu stem rc=$?"
$NCU -i /tmp/${TAG}_stem.ncu-rep --page raw --csv > gpurun_out/${TAG}_stem_raw.csv 2>/dev/null
for k in "conv_tc_kernel<__half, \\(int\\)256, \\(int\\)64" "conv3_nz_kernel<__half, \\(int\\)128"; do
  n=$(echo "$k" | cut -c1-8); $NCU --set full --clock-control none --kernel-name-base demangled -k regex:"$k" --launch-skip 6 -c 1 \
    -o /tmp/${TAG}_$n -f python bench.py --profile-only --no-cpu --no-e2e > /dev/null 2>&1
  $NCU -i /tmp/${TAG}_$n.ncu-rep --page raw --csv > gpurun_out/${TAG}_${n}_raw.csv 2>/dev/null; echo "ncu $n rc=$?"
done
for wl in ${SWEEP:-cfg5_fg95_s512 cfg5_fg95_s384 cfg4_24}; do
  python bench.py --workload $wl --no-cpu --steps 2 > gpurun_out/${TAG}_bench_$wl.json 2> gpurun_out/${TAG}_bench_$wl.err
  echo "$wl rc=$? $(tail -c 300 gpurun_out/${TAG}_bench_$wl.json | head -c 120)"
done
for b in ${BATCHES:-128 256}; do
  python bench.py --workload cfg5_fg95 --batch $b --no-cpu --no-e2e --steps 2 > gpurun_out/${TAG}_bench_cfg5_b$b.json \
    2> gpurun_out/${TAG}_bench_cfg5_b$b.err; echo "batch $b rc=$?"
done
