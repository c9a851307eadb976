cd /root/repo
python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_big.py tests/test_gpu_distributed.py -x -q -m gpu 2>&1 | tail -2
python tools/steptimes.py --config cfg4 --steps 5 --prof 2>&1 | tail -5
