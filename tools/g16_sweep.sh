#!/bin/bash
# k = 16 Jacobi row kernels at cfg4 level 0: threads per row G, unroll U, CTAs per SM, early epilogue operands
cd /root/repo
out=gpurun_out/g16_sweep3.txt; : > $out
for e in 0 1; do
for g in 8:4:8 4:4:4 4:2:5 2:2:4; do
  echo "== BAMG_G16=$g EARLY=$e BAMG_ROWS_PIPE=0" >> $out
  BAMG_EARLY=$e BAMG_G16=$g BAMG_ROWS_PIPE=0 python tools/csr_bench.py --configs cfg4 --ks 16 --reps 6 2>&1 | grep jacobi >> $out
done
done
python - <<'P'
import json
for l in open('gpurun_out/g16_sweep3.txt'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print('   ', d['op'], d['us'], d['frac'])
P
