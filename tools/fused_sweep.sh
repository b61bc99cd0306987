run() { timeout 300 env "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],3), d['config']['zchunk'], d['config']['stages'], d['config']['ctas'])"; }
for st in 3 4 5 6; do echo -n "c2 fused stages=$st: "; run YB_STAGES=$st python bench.py --config c2 --variant fused --steps 20 --warmup 4 --no-cpu-baseline --no-e2e; done
for z in 4 8 16 32 64 128 256; do echo -n "c2 fused z=$z: "; run python bench.py --config c2 --variant fused --zchunk $z --steps 20 --warmup 4 --no-cpu-baseline --no-e2e; done
