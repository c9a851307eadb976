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
    -k regex:"csr_rows|rayleigh_fused_kernel|cgs_dots_kernel|cgs_final_kernel|cgs_update" --csv \
    --log-file gpurun_out/traffic_cfg4.csv python tools/steptimes.py --config cfg4 --steps 1 --prof \
    > gpurun_out/traffic_cfg4_alg.txt 2>&1
echo "traffic rc=$?"
# the two GMRES passes at m ~ 44 (the <32>-group dots and the warp-pair update)
ncu --set full --import-source on --clock-control none -k regex:"cgs_dots_kernel|cgs_update_pair_kernel" -s 62 -c 2 \
    -o gpurun_out/cgs_gram_full -f python tools/steptimes.py --config cfg4 --steps 1 > gpurun_out/cgs_full.log 2>&1
echo "cgs full rc=$?"
# level-0 V-cycle sweeps on the packed operator and the k = 16 smoothing sweep
BAMG_NO_GRAPHS=1 ncu --set full --import-source on --clock-control none -k regex:"csr_rows_stencil1_kernel|csr_rows_packed_kernel" -s 200 -c 3 \
    -o gpurun_out/csr_packed_full -f python tools/steptimes.py --config cfg4 --steps 1 > gpurun_out/csr_packed_full.log 2>&1
echo "packed full rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"csr_rows_stencil_kernel" -c 3 \
    -o gpurun_out/csr_k16_full -f python tools/steptimes.py --config cfg4 --steps 1 > gpurun_out/csr_k16_full.log 2>&1
echo "k16 full rc=$?"
