# A/B of library builds: bench each ab/*.so on the given configs (tb2 variant)
# usage: ABCONF="c2 c3" bash tools/ab_libs.sh
for rep in 1 2; do
for lib in ab/*.so; do for c in ${ABCONF:-c2 c3}; do
  v=$(YB_LIB=$PWD/$lib timeout 300 python bench.py --config $c --variant ${ABVAR:-tb2} --steps 20 --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;print(round(json.loads(sys.stdin.read())['value'],2))")
  echo "$rep $lib $c $v"
done; done; done
# optional: a full checkout of another commit under ab/head (git worktree)
if [ -d ab/head ]; then for rep in 1 2; do for c in ${ABCONF:-c2 c3}; do
  v=$(cd ab/head && timeout 300 python bench.py --config $c --variant ${ABVAR:-tb2} --steps 20 --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;print(round(json.loads(sys.stdin.read())['value'],2))")
  echo "$rep head $c $v"
done; done; fi
