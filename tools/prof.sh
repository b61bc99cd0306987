# one ncu --set full capture of the sweep kernel: PCONF config, PVAR variant, PNAME output name
mkdir -p gpurun_out/p
make -C paper_1301_4539_b200/csrc -j8 >/dev/null 2>&1
C=${PCONF:-c2}; V=${PVAR:-tb2}; N=${PNAME:-prof_${C}_${V}}
K=$(case $V in tb2) echo k_tb2;; tb4) echo k_tb4;; *) echo k_fused;; esac)
CMD="python bench.py --config $C --variant $V --steps 4 --warmup 4 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/p/plain_$N.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s ${PSKIP:-2} -c 1 -o gpurun_out/p/$N $CMD > gpurun_out/p/ncu_$N.log 2>&1; echo ncu=$?
