# Column-block width x z-chunk length (multi-sweep launches), and the TMA maps' L2 promotion with blocks.
one() { # config xblock zchunk [l2promo]
  v=$(YB_TB2_XBLOCK=$2 ${4:+YB_L2PROMO=$4} timeout 300 python bench.py --config $1 --variant tb2 --zchunk $3 --steps 40 --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), d['config']['zchunk'])")
  echo "$1 xblock=$2 zchunk=$3 l2promo=${4:-default} $v"
}
for rep in 1 2; do
  for c in c4 c5; do for w in 0 4; do for z in 64 128 256; do one $c $w $z; done; done; done
  for p in 1 2; do one c4 4 256 $p; one c4 2 256 $p; done
  one c4 3 256; one c4 3 128
done
