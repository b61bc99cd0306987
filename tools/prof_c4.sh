# ncu --set full of one config-4 two-step launch (8 steps = 4 sweeps, MODE 2) + the launch list of
# the default bench command; summaries land in gpurun_out/p4/ (copy to profiles/ to keep).
mkdir -p gpurun_out/p4
O=gpurun_out/p4
CMDP="python bench.py --config c4 --variant tb2 --steps 8 --warmup 4 --no-cpu-baseline --no-e2e"
timeout 300 $CMDP > $O/plain.log 2>&1; echo plain=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tb2 -s 1 -c 1 -o $O/prof_c4_tb2 $CMDP > $O/ncu.log 2>&1; echo ncu=$?
CELLS=$((1024*1024*512*8))
NCU_TRAFFIC_JSON=$O/ncu_traffic.json python tools/ncu_summary.py $O/prof_c4_tb2.ncu-rep c4:tb2 $O/ncu_c4_k_tb2.txt $CELLS > /dev/null 2>&1; echo sum=$?
python tools/ncu_lines.py $O/prof_c4_tb2.ncu-rep 40 > $O/ncu_c4_k_tb2_lines.txt 2>&1; echo lines=$?
ls -la $O
