cd /root/repo
python -m pytest tests/test_gpu_kernels.py -x -q -m gpu 2>&1 | tail -2
echo "== stencil"; python tools/packed_bench.py --config cfg4 --reps 8 2>&1 | tail -4
python tools/steptimes.py --config cfg4 --steps 4 2>&1 | tail -2
python tools/steptimes.py --config cfg1 --steps 6 2>&1 | tail -2
