#!/bin/bash
# ncu --set full captures (with source) of the contiguous half-length DST kernels on the cfg3
# geometry (64 slices): forward (F -> S) and inverse (S -> U) launches.
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:dst_half -c 2 -o gpurun_out/dsthalf -f \
  python tools/profile_heat.py --nt 64 --transform dst --reps 1 > gpurun_out/ncu_dsthalf.log 2>&1
python tools/ncu_summary.py gpurun_out/dsthalf.ncu-rep "contiguous DST pass (forward, inverse), cfg3 geometry, 64 slices" > gpurun_out/contig_summary.txt
python tools/ncu_lines.py gpurun_out/dsthalf.ncu-rep 25 > gpurun_out/contig_lines.txt
head -40 gpurun_out/contig_summary.txt
