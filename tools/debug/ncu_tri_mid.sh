#!/bin/bash
# ncu of the line-solve pass on a mid-size plan (511^2 x 256, 32 tiles: latency-bound, no HBM
# pressure) to see where a step's time goes.
mkdir -p gpurun_out
export STKG_FUSED=1
ncu --set full --clock-control none --import-source on -k regex:heat_tridiag -c 1 -o gpurun_out/trimid -f \
  python tools/profile_heat.py --n 511 --nt 256 --transform dst --reps 1 > gpurun_out/ncu_trimid.log 2>&1
python tools/ncu_summary.py gpurun_out/trimid.ncu-rep "line-solve pass 511^2 x 256" > gpurun_out/trimid_summary.txt
python tools/ncu_lines.py gpurun_out/trimid.ncu-rep 40 > gpurun_out/trimid_lines.txt
tail -12 gpurun_out/trimid_summary.txt
sed -n '/top lines by stall samples/,$p' gpurun_out/trimid_lines.txt | cut -c1-150
