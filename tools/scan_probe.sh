#!/bin/bash
# k3_scan timing of the cfg3 bench for each library build given
for lib in "$@"; do
  echo -n "$lib "
  STKG_LIB_PATH=$PWD/$lib python bench.py --no-alt --no-e2e --no-cpu --no-rksm --no-wave --steps 5 --warmup 3 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', round(d['ms_per_step'],2), 'scan', d['k3_scan'])"
done
