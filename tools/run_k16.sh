cd /root/repo
python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_big.py tests/test_gpu_determinism.py -x -q -m gpu 2>&1 | tail -2
for m in 1 0; do
  echo "== BAMG_NO_STENCIL=$m"
  BAMG_NO_STENCIL=$m python tools/steptimes.py --config cfg4 --steps 5 --prof 2>&1 | tail -5
done
python tools/steptimes.py --config cfg1 --steps 8 2>&1 | tail -3
BAMG_NO_STENCIL=1 python tools/steptimes.py --config cfg1 --steps 8 2>&1 | tail -3
