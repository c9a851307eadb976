#!/bin/bash
# banded coarsest level: width of the subspace block (BAMG_BAND_P = r + guard), cfg4 setup time
cd /root/repo
for p in 32 40 48 56 64; do
  echo "== BAMG_BAND_P=$p"
  BAMG_BAND_P=$p python tools/steptimes.py --config cfg4 --steps 4 2>&1 | grep '"step": 3' | cut -c1-140
done
BAMG_DEBUG=1 python tools/steptimes.py --config cfg4 --steps 1 2>&1 | grep -i "band\|subspace\|ritz" | head -20
