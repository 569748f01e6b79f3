#!/bin/bash
# ncu --set full of KS on chosen layers (args: layer labels)
set -u
mkdir -p gpurun_out
for L in "$@"; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:ks_kernel -s 2 -c 1 \
      -o gpurun_out/ks2_$L python tools/run_layer.py $L 4 > /dev/null 2>&1
  echo "$L rc=$?"
done
