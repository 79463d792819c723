#!/bin/bash
# Builds an experiment variant of libtsg.so with extra nvcc defines (A/B without touching the
# shipped library): tools/build_variant.sh NAME -DFOO=0 ...  ->  paper_1502_00355_b200/libtsg_NAME.so
# Use it with TSG_LIB=paper_1502_00355_b200/libtsg_NAME.so (capi.py).
set -e
name=$1; shift
mkdir -p build/var_$name
NV="nvcc -O3 -std=c++20 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xcompiler -fPIC,-O3 -Iinclude -Ipaper_1502_00355_b200/csrc --expt-relaxed-constexpr $*"
for f in paper_1502_00355_b200/csrc/*.cu; do
  $NV -c $f -o build/var_$name/$(basename $f .cu).o
done
g++ -O3 -std=c++20 -fPIC -Iinclude -Ipaper_1502_00355_b200/csrc $* -c paper_1502_00355_b200/csrc/tsg_prep.cpp -o build/var_$name/tsg_prep.o
nvcc -shared -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xlinker --no-undefined -o paper_1502_00355_b200/libtsg_$name.so build/var_$name/*.o -lpthread
