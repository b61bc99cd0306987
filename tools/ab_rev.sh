# interleaved A/B: the ab/head worktree vs each ab/*.so (env ABENV applied to both)
for c in ${ABCONF:-c3}; do for rep in 1 2; do
  (cd ab/head && env $ABENV timeout 300 python bench.py --config $c --variant tb2 --steps 20 --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null) | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c head', round(d['value'],2))"
  for lib in ab/*.so; do
  env $ABENV YB_LIB=$PWD/$lib timeout 300 python bench.py --config $c --variant tb2 --steps 20 --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c $lib', round(d['value'],2))"
  done
done; done
