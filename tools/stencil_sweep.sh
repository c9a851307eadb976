#!/bin/bash
# k-wide stencil sweeps at cfg4 level 0: CTAs per SM x passes in flight, against the CSR kernels
cd /root/repo
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -x -q -m gpu 2>&1 | tail -2
out=gpurun_out/stencil_sweep.txt; : > $out
for c in 4:2 4:1; do
  echo "== BAMG_STENCIL_CFG=$c" >> $out
  BAMG_STENCIL_CFG=$c python tools/csr_bench.py --configs cfg4 --ks 16 --reps 6 2>&1 | grep -v copy >> $out
done
python - <<'P'
import json
for l in open('gpurun_out/stencil_sweep.txt'):
    if l.startswith('=='): print(l.strip()); continue
    try:
        d=json.loads(l); print('   ', d['op'], d['us'], d['frac'])
    except Exception: print(l.strip()[:200])
P
python tools/steptimes.py --config cfg4 --steps 4 2>&1 | tail -2
