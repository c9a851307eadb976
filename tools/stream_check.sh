#!/bin/bash
# stream-kernel development loop: parity tests, then the level-0 probes
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/stream_tests.log 2>&1; tail -4 gpurun_out/stream_tests.log
for v in 4 6 8 64; do
echo "== BAMG_STREAM_U16=$v"
BAMG_STREAM_U16=$v python tools/smooth_probe.py 2>&1 | head -6
done
python tools/packed_bench.py > gpurun_out/packed_bench_stream.txt 2>&1; tail -7 gpurun_out/packed_bench_stream.txt
python tools/csr_bench.py --configs cfg4 --ks 16 --reps 8 > gpurun_out/csr_bench_stream.txt 2>&1; cat gpurun_out/csr_bench_stream.txt | cut -c1-200
