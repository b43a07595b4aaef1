#!/bin/bash
# Attention phase-trace build (scripts/attn_trace.py): the library with -DPARL_ATTN_TRACE in the
# attention TU, as paper_2511_18871_b200/build/libparl_trace.so (load with PARL_LIB=...).
set -e
cd "$(dirname "$0")/.."
python -m paper_2511_18871_b200._build > /dev/null
B=paper_2511_18871_b200/build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -Iinclude -Ipaper_2511_18871_b200/csrc -DPARL_ATTN_TRACE -c paper_2511_18871_b200/csrc/k_attn_tc.cu -o $B/k_attn_tc_trace.o
objs=$(ls $B/*.o | grep -v k_attn_tc | grep -v trace | grep -v parl_oracle)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $B/libparl_trace.so $objs $B/k_attn_tc_trace.o -lcudart -ldl
echo $B/libparl_trace.so
