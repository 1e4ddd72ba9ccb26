#!/bin/bash
# r4s: bench stall guard: default run through the guard, a forced stall (tiny attempt timeout),
# the self-launched N=2 path, and the reference arm's default invocation untouched
O=gpurun_out/r4s; mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$? lines=$(wc -l < $O/bench.json)" | tee -a $O/status
python -c "import json;d=json.load(open('$O/bench.json'));print(d['value'], d['e2e']['value'], d.get('attempts'), d['cpu_baseline']['value'])"
timeout 300 python bench.py --attempt-timeout 5 > $O/bench_stall.json 2> $O/bench_stall.err; echo "forced-stall rc=$? (expect 1)" | tee -a $O/status; tail -3 $O/bench_stall.err
LP_BENCH_GLOO_TEST=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_n2.json 2> $O/bench_n2.err; echo "bench n2 rc=$?" | tee -a $O/status
python -c "import json;d=json.load(open('$O/bench_n2.json'));print(d['value'], d['n_gpus'])"
