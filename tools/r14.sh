for L in build_ab/lib_d5dc054.so build_ab/lib_e682e3a.so paper_2212_00404_b200/libb200conv.so; do
  echo "== $L"
  B200CONV_LIB_PATH=$PWD/$L timeout 300 python tools/mc_variants.py "B200CONV_REDG=8;B200CONV_REDG=1;B200CONV_SIMT_FORCE=3,43,1;B200CONV_SIMT_FORCE=3,43,1&B200CONV_REDG=1" resnet_14 resnet_7x7 2>&1 | grep fp32
done
