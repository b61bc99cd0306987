# One GPU session: full gpu tests, smoke, bench lines for all configs, reference arm,
# ncu launch list + full captures of the sweep kernels (each ncu command runs
# only after the same command exited 0 without ncu).
mkdir -p gpurun_out/round
O=gpurun_out/round
make -C paper_1301_4539_b200/csrc -j8 >/dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; cat $O/smoke.log
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; echo bench=$?; tail -1 $O/bench_c2.json
for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 20 --warmup 4 > $O/bench_$c.json 2> $O/bench_$c.err; echo $c=$?; done
for c in c1 c2 c3 c4 c5; do timeout 600 python bench.py --config $c --variant fused --steps 20 --warmup 4 --no-cpu-baseline --no-e2e > $O/bench_${c}_fused.json 2> $O/bench_${c}_fused.err; echo ${c}_fused=$?; done
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$?
CMD="python bench.py --steps 4 --warmup 4 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv $CMD > $O/ncu_launch.log 2>&1; echo ncu_launch=$?
for c in c2 c3; do for v in tb2 fused; do
  K=$([ "$v" = tb2 ] && echo k_tb2 || echo k_fused)
  # tb2: warm-up 4 steps = one 2-sweep launch, timed 8 steps = one 4-sweep launch (profiled);
  # fused: one launch per step, the 5th is profiled
  if [ "$v" = tb2 ]; then ST=8; SK=1; else ST=4; SK=4; fi
  CMDP="python bench.py --config $c --variant $v --steps $ST --warmup 4 --no-cpu-baseline --no-e2e"
  timeout 300 $CMDP > $O/plain_${c}_$v.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $SK -c 1 -o $O/prof_${c}_$v $CMDP > $O/ncu_${c}_$v.log 2>&1; echo ncu_${c}_$v=$?
done; done
# summarise on the box (gpurun copies back <= 64 MiB): text summaries + traffic json, keep only
# the config-2 two-step report
cp profiles/ncu_traffic.json $O/ncu_traffic.json
for c in c2 c3; do for v in tb2 fused; do
  k=$([ "$v" = tb2 ] && echo k_tb2 || echo k_fused)
  if [ "$v" = tb2 ]; then ST=8; else ST=1; fi
  CELLS=$(python -c "print({'c2': 256**3, 'c3': 512**3}['$c'] * $ST)")
  NCU_TRAFFIC_JSON=$O/ncu_traffic.json python tools/ncu_summary.py $O/prof_${c}_$v.ncu-rep $c:$v $O/r1_ncu_${c}_${k}.txt $CELLS > /dev/null 2>&1
done; done
python tools/ncu_lines.py $O/prof_c2_tb2.ncu-rep 30 > $O/r1_ncu_c2_k_tb2_lines.txt 2>&1
rm -f $O/prof_c3_*.ncu-rep $O/prof_c2_fused.ncu-rep
du -sh $O

