run() { timeout 300 env "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],3), d['config']['zchunk'], d['config']['stages'])"; }
for z in 16 32 64 128; do for st in 3 4; do echo -n "c3 z=$z st=$st: "; run YB_STAGES=$st python bench.py --config c3 --zchunk $z --steps 20 --warmup 3 --no-cpu-baseline --no-e2e; done; done
for z in 8 16 32; do for st in 3 4 5; do echo -n "c2 z=$z st=$st: "; run YB_STAGES=$st python bench.py --config c2 --zchunk $z --steps 20 --warmup 3 --no-cpu-baseline --no-e2e; done; done
for z in 16 32 64 128 512; do for st in 3 4; do echo -n "c4 z=$z st=$st: "; run YB_STAGES=$st python bench.py --config c4 --zchunk $z --steps 10 --warmup 3 --no-cpu-baseline --no-e2e; done; done
for z in 8 15 32; do for st in 3 4 6; do echo -n "c1 z=$z st=$st: "; run YB_STAGES=$st python bench.py --config c1 --zchunk $z --steps 50 --warmup 3 --no-cpu-baseline --no-e2e; done; done
