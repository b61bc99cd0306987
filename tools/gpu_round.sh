# One GPU session: full gpu tests, smoke, bench lines for all configs, reference arm,
# ncu launch list + full captures of the top kernels.
mkdir -p gpurun_out/round
O=gpurun_out/round
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; cat $O/smoke.log
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; echo bench=$?; tail -1 $O/bench_c2.json
for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 20 --warmup 4 > $O/bench_$c.json 2> $O/bench_$c.err; echo $c=$?; done
for c in c2 c3; do timeout 600 python bench.py --config $c --variant fused --steps 20 --warmup 4 --no-cpu-baseline > $O/bench_${c}_fused.json 2> $O/bench_${c}_fused.err; echo ${c}_fused=$?; done
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$?
CMD="python bench.py --steps 4 --warmup 4 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv $CMD > $O/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tb2 -s 2 -c 1 -o $O/prof_c2_tb2 $CMD > $O/ncu_full.log 2>&1; echo ncu_c2=$?
for v in fused tb2; do
CMD3="python bench.py --config c3 --variant $v --steps 2 --warmup 2 --no-cpu-baseline --no-e2e"
timeout 300 $CMD3 > $O/plain3_$v.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused\|k_tb2 -s 2 -c 1 -o $O/prof_c3_$v $CMD3 > $O/ncu_c3_$v.log 2>&1; echo ncu_c3_$v=$?
done
CMD2="python bench.py --config c2 --variant fused --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD2 > $O/plain2f.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o $O/prof_c2_fused $CMD2 > $O/ncu_c2f.log 2>&1; echo ncu_c2_fused=$?
