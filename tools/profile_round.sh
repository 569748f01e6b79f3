#!/bin/bash
# Round profile capture (run under gpurun from the repo root):
#   1. ncu launch list of one bench step (kernel durations, cold, serialised)
#   2. per-launch DRAM traffic of every hot-path kernel of one step
#   3. one --set full capture of the dominant kernel's heaviest launch
set -u
R=${1:-r01}
mkdir -p gpurun_out
BENCH="python bench.py --steps 2 --warmup 1 --cudnn 0 --cpu-seconds 0 --layers 0 --e2e-steps 1"
K='regex:ks_kernel|kms_kernel|kmtc_kernel|kmtc_persist_kernel|kmn_kernel|splitk_reduce|im2col_kernel|gemm_kernel|pad_kernel|pad_rows_kernel'
NL=$(python -c "import bench; from paper_2212_00404_b200 import conv; print(sum((conv.plan_single(c['Wx'],c['Wy'],c['K'],c['M']) if c['kind']=='single' else conv.plan_multi(c['C'],c['Wx'],c['Wy'],c['K'],c['M'],c['prec']))['launches'] for c in bench.suite()))")
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k "$K" -c $NL --csv --log-file gpurun_out/launches_$R.csv $BENCH \
    > gpurun_out/launches_$R.log 2>&1
echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kms_kernel -s 2 -c 1 \
    -o gpurun_out/full_simt_$R python tools/run_layer.py sweep_14x14_c512_m4096_k3:fp32 3 \
    > /dev/null 2>&1
echo "full rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ks_kernel -s 2 -c 1 \
    -o gpurun_out/full_ks_$R python tools/run_layer.py single_224x224_k1_m256:fp32 3 > /dev/null 2>&1
echo "full ks rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 \
    -o gpurun_out/full_tcg_$R python tools/run_layer.py sweep_14x14_c512_m4096_k3:bf16 3 > /dev/null 2>&1
echo "full tcg rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:kmtc_persist_kernel -s 2 -c 1 \
    -o gpurun_out/full_tcbatched_$R python tools/run_batched.py 64 tf32 3 > /dev/null 2>&1
echo "full tc batched rc=$?"
