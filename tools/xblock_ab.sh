# Item order of multi-sweep launches: column blocks of YB_TB2_XBLOCK tiles (0 = row-major) on the configs in ABCONF.
for rep in 1 2; do for w in ${WIDTHS:-0 1 2 4}; do for c in ${ABCONF:-c4 c5 c3 c2}; do
  v=$(YB_TB2_XBLOCK=$w timeout 300 python bench.py --config $c --variant tb2 --steps ${ABSTEPS:-40} --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), d['clocks']['sm_mhz'])")
  echo "$rep xblock=$w $c $v"
done; done; done
