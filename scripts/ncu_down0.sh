#!/bin/bash
# One full ncu capture of the level-0 stride-2 conv (down0, conv3s2_rc_kernel BN = 64) in the cfg4
# bench command, after a plain run of the same command.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${TAG:-r02d}; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
CMD="python bench.py --profile-only --no-cpu --no-e2e"
$CMD > $O/plain.log 2>&1; echo "plain rc=$?"
$NCU --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"conv3s2_rc_kernel<__half, \(int\)64" -s 20 -c 1 -o $O/down0 -f $CMD > $O/ncu.log 2>&1
echo "ncu rc=$?"
$NCU -i $O/down0.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/down0_raw.csv.gz
$NCU -i $O/down0.ncu-rep --page details 2>/dev/null > $O/down0_details.txt
rm -f $O/down0.ncu-rep
grep -E "Duration|DRAM Throughput|Memory Throughput|Compute \(SM\) Throughput|Issue Slots Busy|Registers Per|Grid Size" $O/down0_details.txt | head -20
