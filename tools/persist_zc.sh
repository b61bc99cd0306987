# persistent multi-sweep launches x z-chunk length
for rep in 1 2; do for cz in "c4 128" "c4 256" "c4 512" "c3 128" "c3 256" "c5 128" "c5 256"; do set -- $cz
  YB_TB2_PERSIST=1 timeout 300 python bench.py --config $1 --zchunk $2 --steps 20 --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$rep $1 z=$2', round(d['value'],2))"
done; done
