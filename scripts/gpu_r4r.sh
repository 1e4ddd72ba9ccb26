#!/bin/bash
# r4r: hunt the intermittent bench stall: repeated default bench runs under a Python stack
# watchdog (120 s), nvidia-smi snapshot while a run is still alive at 100 s
O=gpurun_out/r4r; mkdir -p $O
for rep in $(seq 1 36); do
  LP_WATCH_S=120 python scripts/bench_watch.py --no-cpu-baseline > $O/b_$rep.json 2> $O/b_$rep.err &
  pid=$!
  for t in $(seq 1 130); do
    sleep 1
    kill -0 $pid 2>/dev/null || break
    if [ $t -eq 100 ]; then nvidia-smi > $O/smi_$rep.txt 2>&1; echo "rep $rep still running at 100 s" >> $O/status; fi
  done
  wait $pid; rc=$?
  echo "rep=$rep rc=$rc lines=$(wc -l < $O/b_$rep.json)" >> $O/status
  if [ $rc -ne 0 ]; then echo "rep $rep FAILED" >> $O/status; fi
done
grep -c "rc=0 lines=1" $O/status; grep -v "rc=0 lines=1" $O/status | head
