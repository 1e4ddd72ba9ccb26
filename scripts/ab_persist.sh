echo "== default (non-persistent)"; timeout 300 python -m pytest tests/test_dit_gpu.py -q -x -k "attention or forward" 2>&1 | tail -1
echo "== persistent"; LP_TUNE_ATTN_PERSIST=1 timeout 300 python -m pytest tests/test_dit_gpu.py tests/test_parity_schedule_gpu.py -q -x -k "attention or forward or floor" 2>&1 | tail -1
for v in 0 1 0 1; do echo "persist=$v"; LP_TUNE_ATTN_PERSIST=$v timeout 300 python scripts/kbench.py attn 2>&1 | grep "{" | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); k=list(d)[0]; v=d[k]; print('  ', k, round(v['tflops']))"; done
bash scripts/ab_knob.sh ATTN_PERSIST 0 1
