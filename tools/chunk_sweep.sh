# Multi-sweep two-step launches: z-chunk length vs throughput per config (auto = the built-in model).
one() {  # config zchunk steps
  timeout 300 python bench.py --config $1 --zchunk $2 --steps $3 --warmup 6 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), d['config']['zchunk'])"
}
for rep in 1 2; do
  for z in 4 5 6 7 8 10; do echo "$rep c1 z=$z $(one c1 $z 200)"; done
  for z in 0 12 16 24 32 43 64; do echo "$rep c2 z=$z $(one c2 $z 50)"; done
  for z in 0 32 64 128; do echo "$rep c3 z=$z $(one c3 $z 20)"; done
  for z in 0 32 64 128; do echo "$rep c4 z=$z $(one c4 $z 20)"; done
done
