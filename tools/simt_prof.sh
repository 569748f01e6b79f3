set -u
for L in target_28x28_c256_m256_k3:fp32 alexnet_27x27_c96_m256_k5:fp32 resnet_7x7_c512_m512_k3:fp32; do
  n=${L%%:*}
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:kms_kernel -s 2 -c 1 \
    -o gpurun_out/simt_$n python tools/run_layer.py $L 3 > gpurun_out/simt_$n.log 2>&1
  echo "$L rc=$?"
done
