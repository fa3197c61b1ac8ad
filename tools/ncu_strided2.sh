#!/bin/bash
# A/B of the padded layout with in-place vs out-of-place strided passes, then one
# ncu --set full capture of the 16-byte strided kernel (cfg3 geometry, 64 slices)
mkdir -p gpurun_out
for r in 1 2; do
for oop in 0 1; do echo -n "OOP=$oop "; STKG_PAD_OOP=$oop ./tools/l2chunk_sweep.sh 0; done; done
ncu --set full --clock-control none --import-source on -k regex:dst_half_strided2 -c 1 -o gpurun_out/strided2 -f \
  python tools/profile_heat.py --nt 64 --transform dst --reps 1 > gpurun_out/ncu_strided2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dst_half_strided_kernel -c 1 -o gpurun_out/strided1 -f \
  env STKG_PAD=0 python tools/profile_heat.py --nt 64 --transform dst --reps 1 > gpurun_out/ncu_strided1.log 2>&1
