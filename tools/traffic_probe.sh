# DRAM bytes per cell-update of the sweep kernels for given grids and environment knobs
# usage: TP_GRIDS="1024x1024x512 ..." TP_ENVS="A=1,B=2 ..." TP_VARIANT=tb2 bash tools/traffic_probe.sh
mkdir -p gpurun_out/tp
K=$([ "${TP_VARIANT:-tb2}" = fused ] && echo k_fused || echo k_tb2)
for e in ${TP_ENVS:-none}; do
for n in ${TP_GRIDS:-1024x1024x512}; do
  g=$(echo $n | tr x ' ')
  envs=$([ "$e" = none ] && echo "" || echo $e | tr , ' ')
  env $envs TP_VARIANT=${TP_VARIANT:-tb2} timeout 300 python tools/traffic_probe.py $g > gpurun_out/tp/plain_${n}_$e.log 2>&1
  env $envs TP_VARIANT=${TP_VARIANT:-tb2} timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --print-units base -k regex:$K --csv \
     --log-file gpurun_out/tp/ncu_${n}_$e.csv python tools/traffic_probe.py $g > gpurun_out/tp/ncu_${n}_$e.log 2>&1
  python - $n $e <<'PY'
import csv, sys
n, e = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(f"gpurun_out/tp/ncu_{n}_{e}.csv")) if len(r) > 10 and r[0].isdigit()]
per = {}
for r in rows:
    per.setdefault(int(r[0]), {})[r[-3]] = float(r[-1].replace(",", ""))
x, y, z = (int(v) for v in n.split("x"))
steps = int(open(f"gpurun_out/tp/plain_{n}_{e}.log").read().split(" steps")[0].split()[-1])
# the timed launches: the last ones covering `steps` steps (one launch for multi-sweep, one per sweep/step otherwise)
ids = sorted(per)
rd = sum(per[i]["dram__bytes_read.sum"] for i in ids)
wr = sum(per[i]["dram__bytes_write.sum"] for i in ids)
cu = x * y * z * (steps + 4)
print(n, e, open(f"gpurun_out/tp/plain_{n}_{e}.log").read().strip().split(": ")[-1].split(",")[0],
      "launches %d read B/cu %.2f write B/cu %.2f" % (len(ids), rd / cu, wr / cu))
PY
done; done
