set -x
timeout 400 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench=$?
tail -2 gpurun_out/bench.log
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo c3=$?
tail -1 gpurun_out/bench_c3.log
timeout 300 python bench.py --variant naive --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_naive.log 2>&1; echo naive=$?
tail -1 gpurun_out/bench_naive.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 200 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 4 -c 1 -o gpurun_out/prof_c2 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
tail -3 gpurun_out/ncu_full.log
