# One-step kernel: column-block item order (YB_TB2_XBLOCK; 0 = row-major) on configs 4 / 5 / 3.
for rep in 1 2; do for w in 0 4 2; do for c in c4 c5 c3; do
  v=$(YB_TB2_XBLOCK=$w timeout 300 python bench.py --config $c --variant fused --steps 20 --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],2), round(d['roofline']['frac'],3))")
  echo "fused xblock=$w $c $v"
done; done; done
