# One GPU session: full gpu tests, bench lines for all configs, reference arm,
# ncu launch list + one full capture of the top kernel (c2 default workload).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; cat gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?; tail -1 gpurun_out/bench_c2.json
for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?; done
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?; tail -1 gpurun_out/bench_ref.json
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 4 -c 1 -o gpurun_out/prof_c2 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
CMD3="python bench.py --config c3 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e"
timeout 300 $CMD3 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 1 -o gpurun_out/prof_c3 $CMD3 > gpurun_out/ncu_full3.log 2>&1; echo ncu_full3=$?
