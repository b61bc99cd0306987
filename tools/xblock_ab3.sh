# L2 promotion of the TMA maps (YB_L2PROMO 0 = none, 1 = 64 B, 2 = 128 B, 3 = 256 B) x column-block width x z-chunk.
CONF=${ABCONF:-c4}
for rep in 1 2; do for w in ${WIDTHS:-1 2 4}; do for p in ${PROMOS:-0 1}; do for z in ${CHUNKS:-128 256}; do
  v=$(YB_TB2_XBLOCK=$w YB_L2PROMO=$p timeout 300 python bench.py --config $CONF --variant tb2 --zchunk $z --steps 40 --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2))")
  echo "$CONF xblock=$w l2promo=$p zchunk=$z $v"
done; done; done; done
