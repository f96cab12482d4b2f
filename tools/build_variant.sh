#!/bin/bash
# Build an A/B variant of librs_poly.so with extra nvcc defines (measurement only; the
# product build is paper_1312_5155_b200/_build.py).  Load it with RS_POLY_LIB=<out>.
#   bash tools/build_variant.sh <out.so> -DSOME_MACRO=1
out=$1; shift
C=paper_1312_5155_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
  -diag-suppress 128 -I include -cudart static --threads 0 "$@" -shared -o "$out" \
  $C/rs_kernels.cu $C/polyrs_ablation.cu $C/plan.cpp $C/linear.cpp $C/host_pipeline.cpp $C/jit.cpp -ldl
