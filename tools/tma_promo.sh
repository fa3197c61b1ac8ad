#!/bin/bash
# TMA-staged strided DST pass (STKG_TMA=1) across L2 promotion modes vs the cp.async
# staging: ncu kernel time, DRAM bytes read and L2 read sectors (64-slice cfg3 geometry)
for pr in 0 64 256; do
STKG_TMA=1 STKG_TMA_PROMO=$pr ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:strided -c 2 python tools/profile_heat.py --nt 64 --transform dst --reps 1 2>&1 | grep -E "duration|dram__|lts__" | head -3 | sed "s/^/promo=$pr /"
done
STKG_TMA=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:strided -c 1 python tools/profile_heat.py --nt 64 --transform dst --reps 1 2>&1 | grep -E "duration|dram__|lts__" | sed "s/^/ldgsts /"
