# quick GPU check: parity subset + bench lines for the sweep kernels
mkdir -p gpurun_out/q
make -C paper_1301_4539_b200/csrc -j8 >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x ${QTESTS:+-k "$QTESTS"} > gpurun_out/q/pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/q/pytest.log
for c in ${QCONF:-c2 c3}; do for v in ${QVAR:-tb2 fused}; do
timeout 300 python bench.py --config $c --variant $v --steps 20 --warmup 4 --no-cpu-baseline --no-e2e > gpurun_out/q/b_${c}_$v.json 2>gpurun_out/q/b_${c}_$v.err
python -c "import json;d=json.load(open('gpurun_out/q/b_${c}_$v.json'));print('$c $v', round(d['value'],2), d['roofline']['frac'], d['clocks']['sm_mhz'])"
done; done
