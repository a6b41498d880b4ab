#!/bin/bash
# Precision-budget sweep: per-level plain-storage knobs against the oracle, and
# their per-layer times on cfg4 (under gpurun from the repo root).
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${TAG:-s3}; mkdir -p $O
timeout 900 python scripts/xlevels_parity.py ${PREC_KEYS:-xap=1 plainl=1} > $O/precision.txt 2>&1; echo "precision rc=$?"; cat $O/precision.txt
for k in ${LAYER_KEYS:-none xap=1 plainl=1}; do
  kk=$(echo $k | tr '+' ' '); [ "$k" = none ] && kk=""
  timeout 300 python scripts/layer_profile.py cfg4 fp16f8 2 $kk > $O/layers_$k.txt 2>&1; echo "layers $k rc=$? $(head -1 $O/layers_$k.txt)"
done
