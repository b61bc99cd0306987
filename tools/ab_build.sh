# A/B build of the two-step kernel: ab/<name>.so = the current objects with yb_tb2.cu
# recompiled with extra flags (only the multi-sweep kernels of masks 0 / 2 / 15: -DYB_TB2_AB).
# usage: bash tools/ab_build.sh <name> [extra nvcc flags...]
set -e
name=$1; shift
cd paper_1301_4539_b200/csrc
mkdir -p ../../ab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
  -Xcompiler -fPIC,-ffp-contract=off -Xptxas -v -I../../include -DYB_TB2_AB "$@" \
  -c yb_tb2.cu -o ../../ab/$name.o 2> ../../ab/$name.ptxas.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../ab/$name.so \
  yb_capi.o yb_basic.o yb_fused.o ../../ab/$name.o yb_tb4.o yb_hostops.o yb_xfer.o -Xlinker -lpthread
rm -f ../../ab/$name.o
grep -A2 "k_tb2" ../../ab/$name.ptxas.log | grep -o "k_tb2ILb[01]ELb[01]ELb[01]ELb[01]ELi[0-9]E\|[0-9]* bytes spill stores\|Used [0-9]* registers" | paste - - - 
