#!/bin/bash
# Final round-2 measurement pass (under gpurun from the repo root): bench lines for the
# BASELINE workloads, the cfg4 ncu launch list (conv + front end, DRAM bytes), one full
# source-level capture of the fused-head conv; every ncu command follows a plain run of it.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${TAG:-r02z}; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "bench cfg4 rc=$? $(tail -c 260 $O/bench_cfg4.json | head -c 120)"
for wl in ${WLS:-cfg2 cfg3 cfg4_24 cfg4_paper cfg4_n4 cfg5_fg95 cfg5_fg95_s384 cfg5_fg95_s512}; do
  python bench.py --workload $wl --no-cpu --steps 2 > $O/bench_$wl.json 2> $O/bench_$wl.err; echo "$wl rc=$?"
done
CMD="python bench.py --profile-only --no-cpu --no-e2e"
$CMD > $O/plain.log 2>&1 && \
$NCU --metrics $M --clock-control none --kernel-name-base demangled -k regex:"conv|stem" --launch-skip 200 \
  --launch-count 290 --csv --log-file $O/cfg4_conv.csv $CMD > $O/ncu1.log 2>&1; echo "ncu conv rc=$?"
$NCU --metrics $M --clock-control none --kernel-name-base demangled \
  -k regex:"pyramid|median|hist_kernel|otsu|fg_kernel|tile_keep|compact|finalize|pad_colour|gap_kernel|controller" \
  --launch-count 420 --csv --log-file $O/cfg4_front.csv $CMD > $O/ncu2.log 2>&1; echo "ncu front rc=$?"
$NCU --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"conv3_nz_kernel<__half, \(int\)32, \(int\)8, \(int\)2, \(int\)4" -s 40 -c 1 -o $O/head -f $CMD > $O/ncu3.log 2>&1
echo "ncu head rc=$?"
$NCU -i $O/head.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $O/head_sass.csv.gz
$NCU -i $O/head.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/head_raw.csv.gz
$NCU -i $O/head.ncu-rep --page details 2>/dev/null > $O/head_details.txt
rm -f $O/head.ncu-rep
gzip -f $O/cfg4_conv.csv $O/cfg4_front.csv
ls -la $O
