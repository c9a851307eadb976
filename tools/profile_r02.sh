#!/bin/bash
# Round-2 profiling of the cfg4 headline step on one B200 (run under gpurun).
#   1. ncu launch list of one step (per-launch device time, cold, serialised)
#   2. DRAM traffic of the roofline families over one graph-free step
#   3. --set full captures of the dominant kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv --log-file gpurun_out/launches_cfg4.csv \
    python tools/steptimes.py --config cfg4 --steps 1 > gpurun_out/launches_cfg4.log 2>&1
echo "launch list rc=$?"
BAMG_NO_GRAPHS=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"csr_rows_kernel|rayleigh_fused_kernel|cgs_dots_kernel|cgs_final_kernel" --csv \
    --log-file gpurun_out/traffic_cfg4.csv python tools/steptimes.py --config cfg4 --steps 1 --prof \
    > gpurun_out/traffic_cfg4_alg.txt 2>&1
echo "traffic rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"cgs_dots_kernel" -s 90 -c 2 \
    -o gpurun_out/cgs_dots_full -f python tools/steptimes.py --config cfg4 --steps 1 > gpurun_out/cgs_full.log 2>&1
echo "cgs full rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"cgs_final_kernel" -s 45 -c 1 \
    -o gpurun_out/cgs_final_full -f python tools/steptimes.py --config cfg4 --steps 1 > gpurun_out/cgs_final_full.log 2>&1
echo "cgs final rc=$?"
BAMG_NO_GRAPHS=1 ncu --set full --import-source on --clock-control none -k regex:"csr_rows_kernel" -s 400 -c 3 \
    -o gpurun_out/csr_rows_full -f python tools/steptimes.py --config cfg4 --steps 1 > gpurun_out/csr_full.log 2>&1
echo "csr full rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"bt_sweep_kernel|bt_step_kernel" -s 20 -c 2 \
    -o gpurun_out/band_full -f python tools/steptimes.py --config cfg4 --steps 1 > gpurun_out/band_full.log 2>&1
echo "band full rc=$?"
