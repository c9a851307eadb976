#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over smoke()
# (NOTE: compute-sanitizer is closed on the round-2 GPU pool -- every tool exits 86 there,
# gpurun_out/sanitize_summary.txt; kept for boxes where it is allowed)
# (BASELINE cfg0 through the whole path: setup, dense coarsest, V-cycle graph,
# GMRES) and the band-coarsest pipeline test; logs to gpurun_out/sanitize_*.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
PY='import __graft_entry__ as g; g.smoke()'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python -c "$PY" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool smoke rc=$?" >> gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize_summary.txt
done
timeout 1500 compute-sanitizer --tool memcheck --print-limit 50 --error-exitcode 9 \
  python -m pytest -x -q -m gpu tests/test_gpu_pipeline.py -k "band and uniform63" > gpurun_out/sanitize_band_memcheck.log 2>&1
echo "memcheck band rc=$?" >> gpurun_out/sanitize_summary.txt
tail -3 gpurun_out/sanitize_band_memcheck.log >> gpurun_out/sanitize_summary.txt
timeout 1500 compute-sanitizer --tool racecheck --print-limit 50 --error-exitcode 9 \
  python -m pytest -x -q -m gpu tests/test_gpu_pipeline.py -k "band and uniform63" > gpurun_out/sanitize_band_racecheck.log 2>&1
echo "racecheck band rc=$?" >> gpurun_out/sanitize_summary.txt
tail -3 gpurun_out/sanitize_band_racecheck.log >> gpurun_out/sanitize_summary.txt
