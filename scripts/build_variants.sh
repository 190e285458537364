#!/bin/bash
# Tuning variants of libtilesplat_b200.so (same sources, different -D knobs), built in-tree as
# libtilesplat_b200_<name>.so; load one with TS_LIB_VARIANT=<name>.  usage: build_variants.sh name "FLAGS" ...
cd "$(dirname "$0")/../paper_2602_09999_b200/csrc" || exit 1
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  d=build_$name; mkdir -p $d
  for f in ts_capi k_preprocess k_sort k_blend k_project_bwd k_optim_loss k_loss k_densify k_bin; do
    /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O3 \
      --expt-relaxed-constexpr $flags -c $f.cu -o $d/$f.o &
  done
  wait
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../libtilesplat_b200_$name.so $d/*.o
  echo "built $name ($flags)"
done
