# Temporal-depth sweep on config 5 (1024x1024x256, lossy, 1 GPU):
# d=1 half-step per sweep (naive: E pass, PEC, H pass), d=2 (fused), d=4 (tb2), d=8 (tb4).
mkdir -p gpurun_out/sweep
for v in naive fused tb2 tb4; do
  timeout 600 python bench.py --config c5 --variant $v --steps 12 --warmup 4 --no-cpu-baseline --no-e2e > gpurun_out/sweep/bench_$v.json 2> gpurun_out/sweep/bench_$v.err; echo "$v bench=$?"
done
for v in naive fused tb2 tb4; do
  CMD="python bench.py --config c5 --variant $v --steps 4 --warmup 4 --no-cpu-baseline --no-e2e"
  timeout 300 $CMD > gpurun_out/sweep/plain_$v.log 2>&1 && \
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sweep/ncu_$v.csv $CMD > gpurun_out/sweep/ncu_$v.log 2>&1; echo "$v ncu=$?"
done
