cd /root/repo
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -x -q -m gpu 2>&1 | tail -2
for m in 0 1 2; do
  echo "== BAMG_K16=$m"
  BAMG_K16=$m python tools/steptimes.py --config cfg4 --steps 5 --prof 2>&1 | tail -5
done
