#!/bin/bash
# build the standalone prototype(s) for sm_100a; extra args = -D flags, output name in $OUT
set -e
cd "$(dirname "$0")"
OUT=${OUT:-proto_c2}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xptxas -v "$@" -o $OUT proto_c2.cu 2>&1 | grep -E "error|registers|spill" | grep -B1 -A0 "k_probe_wc\|registers" | grep -E "error|Used" | head -4
