set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "simt_every_tile or (multi_layers_full_size and fp32) or deterministic or graph or multi_edge or multi_integer" > gpurun_out/simt_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/simt_tests.log
for r in 1 2; do
 for L in build_ab/lib_base.so paper_2212_00404_b200/libb200conv.so; do
  echo "== $L" >> gpurun_out/simt_ab.txt
  B200CONV_LIB_PATH=$PWD/$L timeout 300 python tools/mc_variants.py "" resnet vgg_56 alexnet target sweep 2>&1 | grep fp32 >> gpurun_out/simt_ab.txt
 done
done
