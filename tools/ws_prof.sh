# launch list (both kernels) of one layer under a forced KM-SIMT config: ws_prof.sh <layer> <force> <tag>
L=$1; FORCE=$2; TAG=$3
B200CONV_SIMT_FORCE=$FORCE timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:"kms_kernel|splitk" --csv --log-file gpurun_out/ws_$TAG.csv python tools/run_layer.py $L 3 > /dev/null 2>&1
echo "$TAG rc=$?"
