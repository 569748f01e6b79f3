set -u
for prec in tf32 bf16; do for N in 8 32 64; do
  timeout 120 python tools/batched_variants.py "B200CONV_TC_PERSIST=0;B200CONV_TC_PERSIST=1" $N 256 28 3 256 $prec
done; done > gpurun_out/persist1.txt 2>&1
echo "variants rc=$?" >> gpurun_out/persist1.txt
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "batched or padded" >> gpurun_out/persist1.txt 2>&1
echo "tests rc=$?" >> gpurun_out/persist1.txt
