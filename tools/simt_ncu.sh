# ncu --set full of KM-SIMT on one layer with a forced config: simt_ncu.sh <layer> <force> <tag>
L=$1; FORCE=$2; TAG=$3
B200CONV_SIMT_FORCE=$FORCE timeout 300 ncu --set full --clock-control none --import-source on -k regex:kms_kernel -s 2 -c 1 \
  -o gpurun_out/simt_$TAG python tools/run_layer.py $L 3 > gpurun_out/simt_$TAG.log 2>&1
echo "$TAG rc=$?"
