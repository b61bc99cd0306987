# A/B: multi-sweep persistent two-step launches vs one launch per sweep (interleaved, repeated)
make -C paper_1301_4539_b200/csrc -j8 >/dev/null 2>&1
if [ -n "$ABTESTS" ]; then timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/persist_tests.log 2>&1; echo pytest=$?; tail -1 gpurun_out/persist_tests.log; fi
for rep in 1 2; do for c in ${ABCONF:-c1 c2 c3}; do for p in 1 0; do
  YB_TB2_PERSIST=$p timeout 300 python bench.py --config $c --steps ${ABSTEPS:-20} --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$rep $c persist=$p', round(d['value'],2), d['config']['zchunk'], d['roofline']['steps_per_launch'])"
done; done; done
