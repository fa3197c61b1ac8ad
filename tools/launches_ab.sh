#!/bin/bash
# Per-kernel ncu launch times (64-slice cfg3 geometry) of alternative in-tree library builds:
#   tools/launches_ab.sh a.so b.so ...
mkdir -p gpurun_out
for lib in "$@"; do
  STKG_LIB_PATH=$PWD/$lib ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none --csv \
    --log-file gpurun_out/la_$(basename $lib .so).csv python tools/profile_heat.py --nt 64 --transform dst --reps 1 > /dev/null 2>&1
  python - gpurun_out/la_$(basename $lib .so).csv <<'PY'
import csv, sys
rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
agg = {}
for r in rows:
    k = (int(r["ID"]), r["Kernel Name"].split("(")[0][-40:])
    agg.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"])
items = sorted(agg.items())[-7:-2]
print(sys.argv[1], " | ".join(f"{k[1].split('::')[-1]} {v['gpu__time_duration.sum']/1e3:.1f}us {v['l1tex__data_pipe_lsu_wavefronts_mem_shared.sum']/1e6:.1f}M" for k, v in items))
PY
done
