#!/bin/bash
# KS profiling on the 224x224 layers: write-bandwidth probe + ncu full captures
set -u
mkdir -p gpurun_out
python tools/bw_probe.py > gpurun_out/bw_probe.json 2>&1
for L in single_224x224_k1_m256 single_224x224_k3_m256 single_224x224_k7_m256; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:ks_kernel -s 2 -c 1 \
      -o gpurun_out/ks_$L python tools/run_layer.py $L 4 > /dev/null 2>&1
  echo "$L rc=$?"
done
