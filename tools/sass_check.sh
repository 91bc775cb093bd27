#!/bin/bash
# usage: tools/sass_check.sh NT  -> counts shared vs generic memory ops in the solver cubin
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --extended-lambda -Iinclude -Ipaper_1705_06073_b200/csrc \
  -DSLSE_NT=${1:-32} -cubin -o /tmp/s$1.cubin paper_1705_06073_b200/csrc/slse_solve_inst.cu -Xptxas -v 2>&1 | grep -A1 solve_kernel | grep -E "registers|stack"
echo "LDS/STS: $(cuobjdump -sass /tmp/s$1.cubin | grep -c 'LDS\|STS')  generic LD/ST: $(cuobjdump -sass /tmp/s$1.cubin | grep -c 'LD\.E\|ST\.E')"
