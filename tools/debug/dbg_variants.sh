#!/bin/bash
# Build measurement-only variants of the library (global loads / copy-out of the contiguous
# DST kernel removed) to bound what TMA staging could gain.  Run here (nvcc), then time on the GPU.
set -e
mkdir -p variants
cp paper_1912_10082_b200/_stk_gpu.so variants/base.so
for v in NOLDG NOSTG; do
  STKG_NVCC_EXTRA="-DSTKG_DBG_$v" python paper_1912_10082_b200/build.py --force > /dev/null
  cp paper_1912_10082_b200/_stk_gpu.so variants/$v.so
done
cp variants/base.so paper_1912_10082_b200/_stk_gpu.so
touch paper_1912_10082_b200/_stk_gpu.so
