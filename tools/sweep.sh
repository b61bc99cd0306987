for c in c3 c2; do
CMD="python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline --no-e2e"
timeout 200 $CMD > gpurun_out/plain.log 2>&1 || echo FAIL
for st in 2 3 4 5; do
echo "== $c stages=$st"
YB_STAGES=$st timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_sectors_srcunit_tex.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_fused -s 1 -c 1 --csv $CMD 2>/dev/null | grep -E "k_fused" | awk -F'","' '{print $13, $15}'
done; done
