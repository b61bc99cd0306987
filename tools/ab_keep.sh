# A/B of ab/*.so builds (tools/ab_build.sh): full-size oracle parity of c1-c3 through each build,
# then bench lines (kernel only) for the configs in ABCONF, two alternating rounds.
O=gpurun_out/ab
mkdir -p $O
for lib in ${ABLIBS:-ab/*.so}; do
  n=$(basename $lib .so)
  YB_LIB=$PWD/$lib timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -x -k "tb2 and (c1 or c2 or c3)" > $O/parity_$n.log 2>&1
  echo "parity $n rc=$? $(tail -1 $O/parity_$n.log)"
done
for rep in 1 2; do
for lib in ${ABLIBS:-ab/*.so}; do for c in ${ABCONF:-c4 c3 c2}; do
  v=$(YB_LIB=$PWD/$lib timeout 300 python bench.py --config $c --variant tb2 --steps ${ABSTEPS:-20} --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), d['clocks']['sm_mhz'])")
  echo "$rep $lib $c $v"
done; done; done | tee $O/ab.txt
