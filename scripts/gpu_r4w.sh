#!/bin/bash
# r4w: validation of the current build: smoke, all GPU tests, driver-style bench (ours + reference
# arm with its defaults), K1/K10 replay bench and --set full at C2 on all three axes
O=gpurun_out/r4w
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $O/status
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/status
tail -4 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" | tee -a $O/status
python -c "import json;d=json.load(open('$O/bench.json'));print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['step']['frac'], d['clocks']); print(json.dumps(d['hbm_kernels'])[:900])"
HB_TAG=_r4w timeout 600 python scripts/hbm_bench.py 4 > $O/hbm.log 2>&1; mv gpurun_out/hbm_bench_r4w.json $O/hbm_bench.json
HB_NCU=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gather|k_reconstruct" \
   -o $O/hbm_full python scripts/hbm_bench.py 4 > $O/ncu_hbm.log 2>&1; echo "ncu-hbm rc=$?" | tee -a $O/status
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench_ref rc=$?" | tee -a $O/status
cut -c1-600 $O/bench_ref.json
