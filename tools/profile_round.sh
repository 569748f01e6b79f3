#!/bin/bash
# Round profile capture (run under gpurun from the repo root): tools/profile_round.sh <tag>
#   1. ncu launch list of the headline step (configs[4] x FP32/TF32/BF16; cold, serialised)
#   2. --set full captures: KM-SIMT (configs[4] FP32), KM-TC/G GEMM (configs[4] TF32, BF16),
#      KM-TC implicit (28x28x256 N=1 TF32, BF16), KS-L (224x224 K=3 M=256), persistent KM-TC
#      (batched 28x28x256 N=64 TF32, BF16)
#   3. KS DRAM-write evidence: 12 launches of 224x224 K=1 M=256 writing rotating O buffers,
#      --cache-control none (a launch's write-back lands partly in later launches: the
#      per-launch average over the sequence is the DRAM traffic of one launch)
set -u
R=${1:-r02}
mkdir -p gpurun_out
K='regex:ks_kernel|ks_flat_kernel|kms_kernel|kmtc_kernel|kmtc_persist_kernel|kmn_kernel|splitk_reduce|im2col_kernel|gemm_kernel|pad_kernel|pad_rows_kernel'
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k "$K" -c 12 --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 3 --warmup 3 --suite 0 --e2e 0 --cpu-seconds 0 > /dev/null 2>&1
echo "launches rc=$?"
full() {  # full <name> <kernel regex> <layer label> [reps]
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$2" -s 2 -c 1 \
      -o gpurun_out/full_$1_$R python tools/run_layer.py "$3" ${4:-3} > /dev/null 2>&1
  echo "full $1 rc=$?"
}
full simt kms_kernel sweep_14x14_c512_m4096_k3:fp32
full tc4_tf32 kmtc_kernel sweep_14x14_c512_m4096_k3:tf32   # configs[4] TF32 runs on the implicit KM-TC
full tcg_bf16 gemm_kernel sweep_14x14_c512_m4096_k3:bf16
full tc_tf32 kmtc_kernel target_28x28_c256_m256_k3:tf32 4
full tc_bf16 kmtc_kernel target_28x28_c256_m256_k3:bf16 4
full ks3 ks_flat_kernel single_224x224_k3_m256:fp32 4
fullb() {  # fullb <name> <prec>: persistent KM-TC, batched 28x28x256 N=64
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:kmtc_persist -s 1 -c 1 \
      -o gpurun_out/full_$1_$R python tools/run_batched.py 64 $2 3 > /dev/null 2>&1
  echo "full $1 rc=$?"
}
fullb tcp_bf16 bf16
fullb tcp_tf32 tf32
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum --cache-control none \
    --clock-control none -k regex:ks_kernel --csv --log-file gpurun_out/ks_dram_seq_$R.csv \
    python tools/run_layer.py single_224x224_k1_m256:fp32 12 > /dev/null 2>&1
echo "ks dram seq rc=$?"
# KS-L write evidence: 224x224 K=3 M=256 on rotating outputs (L2 write requests / DRAM bytes)
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum,lts__t_requests_op_write.sum,lts__t_sectors_op_write.sum \
    --cache-control none --clock-control none -k regex:ks_ --csv --log-file gpurun_out/ksl_seq_$R.csv \
    python tools/ks_seq.py 224 3 256 12 > /dev/null 2>&1
echo "ksl seq rc=$?"
