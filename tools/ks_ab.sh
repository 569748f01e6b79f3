for L in build_ab/lib_base.so paper_2212_00404_b200/libb200conv.so; do
 echo "== $L"
 B200CONV_LIB_PATH=$PWD/$L timeout 200 python tools/ks_variants.py "" 224 3 32 224 3 64 224 3 128 224 3 256 56 3 256 28 3 256 224 2 64 2>&1 | tail -8
done
