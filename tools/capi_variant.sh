#!/bin/bash
# Build a variant of the C-ABI unit only (slse_capi.cu with extra -D flags),
# linked with the default build's other objects, into build/variants/<name>/.
# Usage: tools/capi_variant.sh <name> [-DFOO=1 ...];  run with SLSE_LIB=build/variants/<name>/libsuperlse_b200.so
cd "$(dirname "$0")/.."
name=$1; shift
out=build/variants/$name
mkdir -p $out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC \
  -Iinclude -Ipaper_1705_06073_b200/csrc "$@" -c paper_1705_06073_b200/csrc/slse_capi.cu -o $out/slse_capi.o || exit 1
objs=$(ls build/obj/*.o | grep -v slse_capi.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $out/libsuperlse_b200.so $out/slse_capi.o $objs
cuobjdump --dump-resource-usage $out/slse_capi.o 2>/dev/null | grep -A1 'grid_r3' | grep -o 'r3_kernelILi[0-9]\|REG:[0-9]*\|STACK:[0-9]*' | paste - - -
