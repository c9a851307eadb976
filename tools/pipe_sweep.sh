#!/bin/bash
cd /root/repo
python -m pytest tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/pipe_kernels_test.log 2>&1; tail -2 gpurun_out/pipe_kernels_test.log
out=gpurun_out/pipe_sweep.txt; : > $out
for cfg in 0 16:6:3 16:5:4 16:4:5 16:4:4 16:6:4 16:8:3; do
  echo "== BAMG_ROWS_PIPE=$cfg" >> $out
  BAMG_ROWS_PIPE=$cfg python tools/csr_bench.py --configs cfg4 --ks 16 --reps 8 >> $out 2>&1
done
for cfg in 0 1:8:4 1:8:6 1:6:6 1:6:5 1:4:6 1:4:8; do
  echo "== BAMG_ROWS_PIPE=$cfg" >> $out
  BAMG_ROWS_PIPE=$cfg python tools/csr_bench.py --configs cfg4 --ks 1 --reps 8 >> $out 2>&1
done
