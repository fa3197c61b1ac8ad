#!/bin/bash
# ncu --set full capture (with source) of the line-solve axis-0 pass on the full cfg3 solve
# (one 1024-slice launch: the overlapped schedule is off under STKG_OVERLAP=0) and of the
# contiguous transform pass beside it, summarised per kernel and per source line.
mkdir -p gpurun_out
export STKG_OVERLAP=0
python tools/solve_time.py --cfg cfg3 --reps 1 > gpurun_out/tri_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:heat_tridiag -c 1 -o gpurun_out/tri -f \
  python tools/solve_time.py --cfg cfg3 --reps 1 > gpurun_out/ncu_tri.log 2>&1
python tools/ncu_summary.py gpurun_out/tri.ncu-rep "line-solve axis-0 pass, cfg3 (1023^2 x 1024), one launch" > gpurun_out/tri_summary.txt
python tools/ncu_lines.py gpurun_out/tri.ncu-rep 25 > gpurun_out/tri_lines.txt
tail -30 gpurun_out/tri_summary.txt
