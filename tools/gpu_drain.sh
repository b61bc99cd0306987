# Streamed readback (yb_run_to_host): its GPU tests, then the default bench line (e2e streamed vs readback after run).
O=gpurun_out/drain
mkdir -p $O
timeout 600 python -m pytest tests/test_run_to_host_gpu.py tests/test_abi.py -q -x > $O/pytest.log 2>&1; echo pytest=$?; tail -15 $O/pytest.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo bench=$?; tail -c 1500 $O/bench_c4.json; tail -5 $O/bench_c4.err
