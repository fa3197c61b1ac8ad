#!/bin/bash
# The round's bench evidence: default bench line (skipped with "ncu"), then the ncu launch
# list of the same solve (per-launch time and DRAM bytes; cold-cache, serialised -- shares,
# not absolutes).  The side legs (wave PCG: thousands of launches) stay out of the capture.
mkdir -p gpurun_out
[ "$1" == "ncu" ] || { timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -c 400 gpurun_out/bench.log; echo; }
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 200 --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 1 --warmup 3 --no-alt --no-e2e --no-cpu --no-rksm --no-wave --no-cn \
  > gpurun_out/ncu_bench.log 2>&1; echo ncu_rc=$?
