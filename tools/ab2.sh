run() { timeout 300 env "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],3), d['config']['zchunk'], d['config']['stages'])"; }
for t in 1 2 3; do echo -n "c2 fused: "; run python bench.py --config c2 --steps 20 --warmup 4 --no-cpu-baseline --no-e2e; done
echo -n "c2 fused st3: "; run YB_STAGES=3 python bench.py --config c2 --steps 20 --warmup 4 --no-cpu-baseline --no-e2e
echo -n "c2 fused z8: "; run python bench.py --config c2 --zchunk 8 --steps 20 --warmup 4 --no-cpu-baseline --no-e2e
echo -n "c2 fused z32: "; run python bench.py --config c2 --zchunk 32 --steps 20 --warmup 4 --no-cpu-baseline --no-e2e
CMD="python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 200 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 4 -c 1 -o gpurun_out/prof_c2_f2 $CMD > gpurun_out/ncu.log 2>&1; echo ncu=$?
