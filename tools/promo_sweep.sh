#!/bin/bash
# DRAM traffic of the C4 GEMMs vs the TMA L2 promotion (CK_TMA_PROMO).  gpurun_out/promo_p<P>.csv
set -u
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_op_read_hit_rate.pct,sm__cycles_elapsed.avg.per_second"
for P in "${@:-0 2 3}"; do
  CK_TMA_PROMO=$P timeout 600 ncu --metrics "$M" --clock-control none -k regex:gemm_bf16x3 --launch-skip 3 --launch-count 3 \
    --csv --log-file gpurun_out/promo_p$P.csv python tools/profile_step.py 32768 4096 4096 8 32768 > /dev/null 2>&1
  echo "promo $P rc=$?"
done
