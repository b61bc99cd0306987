# Depth of the tail skew (YB_DRAIN_K) of the one-call streamed flow on config 4 (stream_phases prints the e2e times).
for k in ${KS:-32 40 48 56}; do
  echo "K=$k $(YB_DRAIN_K=$k NX=1024 NY=1024 NZ=512 STEPS=200 CELLS=1 FIELDS=0 python tools/stream_phases.py 2>&1 | grep 'run_streamed(200)' | sed 's/.*run_streamed(200): //' | cut -c1-40 | tr '\n' '|')"
done
