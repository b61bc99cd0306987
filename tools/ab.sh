timeout 300 python tools/tb2_check.py 2>&1 | tail -2
run() { timeout 300 env "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],3), d['roofline']['algorithmic_bytes_per_cell_update'], d['config']['zchunk'], d['config']['stages'], round(d['roofline']['step_ms_share_of_kernel'],3))"; }
for c in c1 c2 c3 c4 c5; do for v in fused tb2; do echo -n "$c $v: "; run python bench.py --config $c --variant $v --steps 20 --warmup 4 --no-cpu-baseline --no-e2e; done; done
for z in 32 64 128; do echo -n "c3 tb2 z=$z: "; run python bench.py --config c3 --variant tb2 --zchunk $z --steps 20 --warmup 4 --no-cpu-baseline --no-e2e; done
CMD="python bench.py --config c3 --variant tb2 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e"
timeout 200 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tb2 -s 1 -c 1 -o gpurun_out/prof_c3_tb2b $CMD > gpurun_out/ncu_tb2.log 2>&1; echo ncu=$?
