#!/bin/bash
# k = 1 row kernel on the Galerkin levels of the V-cycle: unroll x CTAs per SM x early operands
cd /root/repo
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -x -q -m gpu 2>&1 | tail -1
for c in 0 8:5:1 8:6:1 8:6:0; do
  echo "== BAMG_K1W=$c"
  BAMG_K1W=$c python tools/steptimes.py --config cfg4 --steps 3 2>&1 | grep '"step": 2' | cut -c1-140
done
