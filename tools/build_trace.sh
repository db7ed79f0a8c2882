#!/bin/sh
# debug build of libneob200 with CTA-0 event tracing (tools/trace_conv.py)
cd "$(dirname "$0")/../paper_1809_02697_b200/csrc" && \
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DNEO_TRACE -Xcompiler -fPIC -shared \
     -o ../../tools/libneob200_trace.so abi.cu conv_tc.cu conv_simt.cu layout.cu ops.cu stem.cu head.cu
