set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "tc_paths or strided or multi_layers or shard or deterministic or graph" > gpurun_out/gemm_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gemm_tests.log
for r in 1 2; do
 for L in build_ab/lib_base.so paper_2212_00404_b200/libb200conv.so; do
  echo "== $L" >> gpurun_out/gemm_ab.txt
  B200CONV_LIB_PATH=$PWD/$L timeout 300 python tools/mc_variants.py "" sweep resnet_7x7 2>&1 | grep -v fp32 >> gpurun_out/gemm_ab.txt
 done
done
