#!/bin/bash
# ncu --set full captures (with source) of the half-length DST kernels on the cfg3 geometry
# (64 slices).
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:dst_half -c 2 -o gpurun_out/dsthalf -f \
  python tools/profile_heat.py --nt 64 --transform dst --reps 1 > gpurun_out/ncu_dsthalf.log 2>&1
