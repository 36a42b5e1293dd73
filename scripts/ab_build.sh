#!/bin/bash
# Build the CUDA library from a git revision (or the working tree: "wt") into build/ab/<name>/
# for A/B timing: CSPQ_LIB_PATH=build/ab/<name>/libcspq_b200.so python scripts/probe_tc_bits.py ...
# NVFLAGS="-DCSPQ_TC_PROBES -DCSPQ_TC_STAMPS" builds the instrumented kernel (probe bits, clock stamps).
set -e
rev=$1; name=$2
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/build/ab/$name
mkdir -p "$out"
if [ "$rev" = wt ]; then src=$root/paper_2605_25521_b200/csrc; else
  src=$(mktemp -d); git -C "$root" archive "$rev" paper_2605_25521_b200/csrc include | tar -x -C "$src"; src=$src/paper_2605_25521_b200/csrc; fi
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --ftz=false \
  --prec-div=true --prec-sqrt=true ${NVFLAGS:-} -shared -o "$out/libcspq_b200.so" $src/encode.cu $src/encode_tc.cu $src/lloyd.cu \
  $src/fileio.cu $src/adc.cu $src/capi.cu -lcudart
echo "$out/libcspq_b200.so"
