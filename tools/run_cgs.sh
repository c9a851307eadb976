cd /root/repo
python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_big.py tests/test_gpu_distributed.py -x -q -m gpu 2>&1 | tail -2
for mid in 0 1; do
echo "== BAMG_CGS_MID=$mid"
BAMG_CGS_MID=$mid python tools/steptimes.py --config cfg4 --steps 5 --prof 2>&1 | tail -5 | grep -E "step|gmres_cgs"
done
python tools/steptimes.py --config cfg2 --steps 6 --prof 2>&1 | tail -5 | grep -E "step|gmres_cgs"
