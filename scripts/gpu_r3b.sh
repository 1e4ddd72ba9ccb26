#!/bin/bash
# r3b: HBM-kernel evidence (replay bench + ncu --set full on K1/K10 per C2 axis), bench with the
# replay-timed hbm section, compute-sanitizer pass.
O=gpurun_out/r3b
mkdir -p $O
timeout 600 python scripts/hbm_bench.py 4 > $O/hbm_bench.log 2>&1; echo "hbm rc=$?" | tee -a $O/status
mv gpurun_out/hbm_bench.json $O/ 2>/dev/null; cat $O/hbm_bench.log | cut -c1-400
HB_NCU=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gather_entries|k_reconstruct" \
   -o $O/hbm_full python scripts/hbm_bench.py 4 > $O/ncu_hbm.log 2>&1; echo "ncu-hbm rc=$?" | tee -a $O/status
tail -3 $O/ncu_hbm.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" | tee -a $O/status
python -c "import json;d=json.load(open('$O/bench.json'));print(d['value'], json.dumps(d['hbm_kernels'])[:1500])"
bash scripts/sanitize.sh $O/sanitize
