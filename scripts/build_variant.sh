#!/bin/bash
# Build a libhmf.so variant with extra -D flags on the Q-band translation unit
# (A/B experiments on the GPU box): build/var/NAME/libhmf.so.  Swap it into
# paper_2006_15980_b200/lib/ for a run, then restore the default build.
#   scripts/build_variant.sh NAME -DRUNS_LPC_256=8 -DRUNS_WPB_256=8
set -e
NAME=$1; shift
D=build/var/$NAME; mkdir -p $D
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC \
  -I include "$@" -c -o $D/qband_kernels.o paper_2006_15980_b200/csrc/qband_kernels.cu
objs=$(ls build/obj/*.o | grep -v qband_kernels.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xcompiler -fPIC \
  -o $D/libhmf.so $D/qband_kernels.o $objs -lrt
echo $D/libhmf.so
