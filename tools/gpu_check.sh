# Health check of HEAD on one B200: GPU tests, smoke, default bench line.
O=gpurun_out/check
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $O/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; cat $O/smoke.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo bench=$?; tail -c 600 $O/bench_c4.json
