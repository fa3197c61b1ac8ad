#!/bin/bash
# ncu launch lists (time, DRAM bytes) of the cfg3-geometry DST solve, padded vs unpadded layout
mkdir -p gpurun_out
for pad in 1 0; do
STKG_PAD=$pad ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum --clock-control none --csv \
  --log-file gpurun_out/launches_pad$pad.csv python tools/profile_heat.py --nt 64 --transform dst --reps 1 > gpurun_out/launches_pad$pad.log 2>&1
done
