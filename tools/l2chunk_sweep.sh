#!/bin/bash
# Sweep the L2 sub-chunk budget of the device heat solve (STKG_L2_CHUNK_MB) on cfg3.
for mb in "$@"; do
  STKG_L2_CHUNK_MB=$mb python bench.py --no-alt --no-e2e --no-cpu --no-rksm --steps 5 --warmup 3 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('MB', $mb, 'ms/step', round(d['ms_per_step'],2), 'value', '%.3e' % d['value'], 'launches', d['gpu_launches'], 'dst GB/s', round(d['roofline']['achieved']), 'relres', d['config']['relres_gpu_k1'])"
done
