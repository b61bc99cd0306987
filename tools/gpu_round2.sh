# Round-2 GPU session: full GPU tests, smoke, bench lines (config 4 default + the others),
# the reference arm, the ncu launch list of the default bench command and one ncu --set full
# capture of the config-4 two-step kernel. Output: gpurun_out/round2/ (summaries to copy into profiles/).
O=gpurun_out/round2
mkdir -p $O
make -C paper_1301_4539_b200/csrc -j8 >/dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; cat $O/smoke.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo bench=$?
for c in c1 c2 c3 c5; do timeout 600 python bench.py --config $c --steps 20 --warmup 4 > $O/bench_$c.json 2> $O/bench_$c.err; echo $c=$?; done
timeout 600 python bench.py --variant fused --steps 20 --warmup 4 --no-cpu-baseline --no-e2e > $O/bench_c4_fused.json 2> $O/bench_c4_fused.err; echo c4_fused=$?
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$?
CMD="python bench.py --steps 10 --warmup 4 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv $CMD > $O/ncu_launch.log 2>&1; echo ncu_launch=$?
CMDP="python bench.py --config c4 --variant tb2 --steps 8 --warmup 4 --no-cpu-baseline --no-e2e"
timeout 300 $CMDP > $O/plain_p.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tb2 -s 1 -c 1 -o $O/prof_c4_tb2 $CMDP > $O/ncu_full.log 2>&1; echo ncu_full=$?
NCU_TRAFFIC_JSON=$O/ncu_traffic.json python tools/ncu_summary.py $O/prof_c4_tb2.ncu-rep c4:tb2 $O/r2_ncu_c4_k_tb2.txt $((1024*1024*512*8)) > /dev/null 2>&1
python tools/ncu_lines.py $O/prof_c4_tb2.ncu-rep 40 > $O/r2_ncu_c4_k_tb2_lines.txt 2>&1
for f in $O/bench_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', d.get('value'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'))" 2>/dev/null; done
du -sh $O
