#!/bin/bash
# Dev: build paper_2307_05590_b200/libpodp_<name>.so with k_lu_ll.cu compiled under extra defines.
#   tools/devlib.sh <name> "-DPODP_LL_ABLATE=1 -DPODP_LL_G=8"
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2307_05590_b200 import _build; _build.build()"
B=paper_2307_05590_b200/build
OBJS=$(ls $B/*.o | grep -v k_lu_ll)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC,-O2 \
  --expt-relaxed-constexpr -I include -I paper_2307_05590_b200/csrc $2 \
  -c paper_2307_05590_b200/csrc/k_lu_ll.cu -o /tmp/ll_$1.o -Xptxas -v 2>&1 \
  | grep -A2 "${KFILT:-lu_ll_kernelILi48ELb1ELb0ELb1ELb0}" | grep -E "registers|spill" || true
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
  -o paper_2307_05590_b200/libpodp_$1.so $OBJS /tmp/ll_$1.o -cudart static
