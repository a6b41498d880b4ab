#!/bin/bash
# Full ncu capture (source-level) of the fused-head conv on a 40x (one-task) batch of cfg4.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${TAG:-s4}; mkdir -p $O
CMD="python bench.py --profile-only --no-cpu --no-e2e $EXTRA"
$CMD > $O/plain.log 2>&1 && \
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"${KREGEX:-conv3_nz_kernel<__half, \(int\)32, \(int\)8, \(int\)2, \(int\)4}" -s ${SKIP:-40} -c 1 \
  -o $O/head -f $CMD > $O/ncu.log 2>&1; echo "ncu rc=$?"
# the report itself exceeds gpurun's copy-back limit: export text views and drop it
N=/usr/local/cuda/bin/ncu
$N -i $O/head.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $O/head_sass.csv.gz
$N -i $O/head.ncu-rep --page source --csv --print-source cuda 2>/dev/null | gzip > $O/head_cuda.csv.gz
$N -i $O/head.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/head_raw.csv.gz
$N -i $O/head.ncu-rep --page details 2>/dev/null > $O/head_details.txt
rm -f $O/head.ncu-rep; ls -la $O
