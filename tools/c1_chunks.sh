# Config 1 (128^3, L2-resident): one launch per sweep vs multi-sweep launches at forced z-chunks.
for rep in 1 2; do
  v=$(YB_TB2_PERSIST=0 timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), d['config']['zchunk'])")
  echo "$rep single-sweep $v"
  for z in 8 12 16 24 32 43 64 128; do
    v=$(timeout 300 python bench.py --config c1 --zchunk $z --steps 200 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), d['config']['zchunk'], d['roofline']['steps_per_launch'] if 'steps_per_launch' in d['roofline'] else '')")
    echo "$rep z=$z $v"
  done
done
