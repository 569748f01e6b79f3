set -u
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "persistent or batched" > gpurun_out/sk_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/sk_tests.log
for prec in tf32 bf16; do for N in 32 64; do
  timeout 120 python tools/batched_variants.py "B200CONV_TC_STREAMK=0;B200CONV_TC_STREAMK=1" $N 256 28 3 256 $prec
done; done > gpurun_out/sk_ab.txt 2>&1
echo "ab rc=$?" >> gpurun_out/sk_ab.txt
