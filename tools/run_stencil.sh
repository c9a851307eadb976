cd /root/repo
python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "packed or pack" 2>&1 | tail -3
echo "== stencil"; python tools/packed_bench.py --config cfg4 --reps 8 2>&1 | tail -7
echo "== no stencil"; BAMG_NO_STENCIL=1 python tools/packed_bench.py --config cfg4 --reps 8 2>&1 | tail -4
python tools/steptimes.py --config cfg4 --steps 4 2>&1 | tail -2
