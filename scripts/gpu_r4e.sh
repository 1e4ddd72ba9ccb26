#!/bin/bash
# r4e: stress the CTA-pair attention (an r4d bench run with ring depths 3/3 printed nothing)
O=gpurun_out/r4e; mkdir -p $O
P=paper_2512_07350_b200/liblp_b200.so; cp $P /tmp/orig.so
for v in p33 p44; do
  cp ab/liblp_$v.so $P
  for rep in 1 2 3; do
    LP_TUNE_ATTN_PAIR=1 timeout 600 python bench.py --no-cpu-baseline --steps 6 --warmup 3 > $O/bench_${v}_$rep.json 2> $O/bench_${v}_$rep.err
    echo "$v rep=$rep rc=$? $(tail -c 300 $O/bench_${v}_$rep.err | tr '\n' ' ' | cut -c1-300)" | tee -a $O/status
  done
  LP_TUNE_ATTN_PAIR=1 timeout 600 python -m pytest -m gpu -q -p no:cacheprovider tests/test_dit_gpu.py -k "attention or forward" > $O/pytest_$v.log 2>&1
  echo "$v tests rc=$? $(tail -1 $O/pytest_$v.log)" | tee -a $O/status
done
cp /tmp/orig.so $P
