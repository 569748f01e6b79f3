# time multi-channel bench layers under several library builds: ab_libs.sh <label-substr...>  (libs: build_ab/lib_*.so + current)
for L in build_ab/lib_*.so paper_2212_00404_b200/libb200conv.so; do
  echo "== $L"
  B200CONV_LIB_PATH=$PWD/$L timeout 300 python tools/mc_variants.py "" "$@" 2>&1 | grep fp32
done
