# Streamed upload (yb_run_streamed): e2e of the configs named in CONFS (default c4 c3 c5 c2) with the three
# flows bench.py reports (one call / upload then run_to_host / phase by phase), kernel line included.
O=gpurun_out/stream
mkdir -p $O
for c in ${CONFS:-c4 c3 c5 c2}; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
  python - <<PY
import json
d=json.loads(open('$O/bench_$c.json').read().strip().splitlines()[-1])
e=d['e2e']
print('$c', 'value', round(d['value'],1), 'e2e', round(e['value'],1), 'wall', round(e['wall_s'],4),
      'upload_then', round(e.get('upload_then_run_to_host',{}).get('value',0),1),
      'phases', round(e.get('readback_after_run',{}).get('value',0),1))
PY
done
