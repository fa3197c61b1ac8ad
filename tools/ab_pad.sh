#!/bin/bash
# GPU heat tests, then A/B of the cfg3 solve with the padded internal layout on / off
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_heat_gpu.py -x -q > gpurun_out/heat_tests.log 2>&1; echo rc=$? >> gpurun_out/heat_tests.log
tail -3 gpurun_out/heat_tests.log
for r in 1 2; do
for pad in 1 0; do
echo -n "PAD=$pad "; STKG_PAD=$pad ./tools/l2chunk_sweep.sh 0
done; done
