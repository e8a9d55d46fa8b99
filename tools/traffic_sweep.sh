#!/bin/bash
# DRAM / L2 traffic of the C4 GEMMs (one 32768-row chunk) vs the rasterisation
# group (dev tool; run on the GPU box).  Writes gpurun_out/traffic_g<G>.csv.
#   bash tools/traffic_sweep.sh [groups...]
set -u
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_op_read_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active"
for G in "${@:-1 2 4 8 16 32}"; do
  CK_GEMM_GROUP=$G timeout 600 ncu --metrics "$M" --clock-control none -k regex:gemm_bf16x3 --launch-skip 3 --launch-count 3 \
    --csv --log-file gpurun_out/traffic_g$G.csv python tools/profile_step.py 32768 4096 4096 8 32768 > /dev/null 2>&1
  echo "group $G rc=$?"
done
