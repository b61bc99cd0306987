# Measurement build ab/stamp.so: per-item timestamps of the multi-sweep two-step launch
# (-DYB_TB2_STAMP; written to $YB_TB2_STAMP_FILE by every multi-sweep launch). See tools/stamp_drift.py.
set -e
cd paper_1301_4539_b200/csrc
mkdir -p ../../ab
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC,-ffp-contract=off -I../../include -DYB_TB2_AB -DYB_TB2_STAMP"
nvcc $F -c yb_tb2.cu -o ../../ab/stamp_tb2.o &
nvcc $F -c yb_capi.cu -o ../../ab/stamp_capi.o &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../ab/stamp.so ../../ab/stamp_capi.o yb_basic.o yb_fused.o ../../ab/stamp_tb2.o yb_tb4.o yb_hostops.o yb_xfer.o -Xlinker -lpthread
rm -f ../../ab/stamp_*.o
