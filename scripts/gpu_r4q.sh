#!/bin/bash
# r4q: bench robustness — repeated default bench runs with stderr kept (two A/B runs printed no line)
O=gpurun_out/r4q; mkdir -p $O
for rep in 1 2 3 4 5 6 7 8; do
  timeout 600 python bench.py --no-cpu-baseline > $O/bench_$rep.json 2> $O/bench_$rep.err
  rc=$?
  echo "rep=$rep rc=$rc lines=$(wc -l < $O/bench_$rep.json) $(tail -c 400 $O/bench_$rep.err | tr '\n' ' ')" | tee -a $O/status
done
