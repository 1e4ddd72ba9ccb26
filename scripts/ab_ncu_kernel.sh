#!/bin/bash
# Per-variant ncu launch times of one kernel inside a short bench run.
# usage: bash scripts/ab_ncu_kernel.sh KERNEL_REGEX "FLAGS_A" "FLAGS_B" ...
K=$1; shift
for f in "$@"; do
  LP_NVCC_EXTRA="$f" python -c "from paper_2512_07350_b200 import build; build.build()" > /dev/null
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$K -c 120 --csv \
      python bench.py --steps 1 --warmup 1 --no-cpu-baseline --layers 4 2>/dev/null | python -c "
import csv, sys
rows = [r for r in csv.reader(l for l in sys.stdin if l.startswith('\"'))]
h = rows[0]; v = [float(r[h.index('Metric Value')]) for r in rows[1:]]
u = rows[1][h.index('Metric Unit')]
print('[$f]', len(v), 'launches, mean', round(sum(v) / len(v), 2), u)"
done
python -c "from paper_2512_07350_b200 import build; build.build()" > /dev/null
