cd /root/repo
python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_big.py tests/test_gpu_kernels.py -x -q -m gpu 2>&1 | tail -1
BAMG_NVTX=0 python tools/breakdown.py --config cfg4 --reps 2 --top 12 2>&1 | grep -E "rayleigh|TRACE|stencil_kernel"
python tools/steptimes.py --config cfg4 --steps 4 --prof 2>&1 | tail -5 | cut -c1-150
