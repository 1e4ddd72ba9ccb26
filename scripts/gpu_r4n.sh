#!/bin/bash
# r4n: bench with the step graphs primed before the warm-up: N=1 (x2), the self-launched N=2 on one GPU
O=gpurun_out/r4n; mkdir -p $O
for rep in 1 2; do
timeout 900 python bench.py --no-cpu-baseline > $O/bench_$rep.json 2> $O/bench_$rep.err; echo "bench rc=$?" | tee -a $O/status
python -c "import json;d=json.load(open('$O/bench_$rep.json'));print(d['value'], d['e2e']['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['step']['frac'])"
done
LP_BENCH_GLOO_TEST=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_n2.json 2> $O/bench_n2.err; echo "bench n2 rc=$?" | tee -a $O/status
python -c "import json;d=json.load(open('$O/bench_n2.json'));print(d['value'], d['n_gpus'], d['exchange'])"
timeout 900 python -m pytest -m gpu -q -p no:cacheprovider tests/test_bench_multirank_gpu.py > $O/pytest_bench.log 2>&1; echo "bench tests rc=$?" | tee -a $O/status; tail -1 $O/pytest_bench.log
