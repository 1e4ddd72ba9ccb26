#!/bin/bash
# r3k: what the LN fold costs — interleaved C2 bench: no fold | fold | fold without the xq
# stores | fold without xq stores and partials (the last two give wrong numbers: timing only).
# Also validates the graph-replayed lp_engine_hbm_bench inside bench.py.
O=gpurun_out/r3k; mkdir -p $O
P=paper_2512_07350_b200/liblp_b200.so
cp $P $O/.orig.so
run() { timeout 600 env LP_TUNE_DIT_LNFOLD=$2 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', json.dumps({'value': round(d['value'],4), 'sm_mhz': d['clocks']['sm_mhz'], 'tflops': {k: round(v['tflops']) for k, v in d['kernels'].items()}, 'k1': round(d['hbm_kernels']['k1_gather']['frac_of_hbm'],3), 'k10': {a: round(v['frac_of_hbm'],2) for a,v in d['hbm_kernels']['k10_reconstruct_update']['per_axis'].items()}}))"; }
for rep in 1 2; do
  cp ab/liblp_base.so $P; run nofold 0; run fold 1
  cp ab/liblp_noxq.so $P; run fold_noxq 1
  cp ab/liblp_noxqm.so $P; run fold_noxq_nomerge 1
done 2>&1 | tee $O/ab.txt
cp $O/.orig.so $P && rm $O/.orig.so
