#!/bin/bash
# Build an A/B variant of libtkb.so with extra -D flags: tools/build_variant.sh NAME "-DFOO=1 ..."
# Output: build/libtkb_NAME.so (load with TKB_LIB_PATH=build/libtkb_NAME.so).
set -e
cd "$(dirname "$0")/../paper_2410_20399_b200/csrc"
mkdir -p ../../build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I. -I../../include -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr $2 -shared capi.cu attn_fwd_sm100.cu attn_bwd_sm100.cu \
    rotary_sm100.cu gemm_sm100.cu util_kernels.cu -o ../../build/libtkb_$1.so
