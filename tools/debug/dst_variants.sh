#!/bin/bash
# Build tuning variants of the contiguous DST kernel (compile-time knobs) for an A/B on the GPU.
set -e
mkdir -p variants
cp paper_1912_10082_b200/_stk_gpu.so variants/base.so
build() { STKG_NVCC_EXTRA="$2" python paper_1912_10082_b200/build.py --force > /dev/null; cp paper_1912_10082_b200/_stk_gpu.so variants/$1.so; }
build pf2 "-DSTKG_DST_PREFETCH=2"
build pf0 "-DSTKG_DST_PREFETCH=0"
build mb6 "-DSTKG_HALF_MINB=6"
build mb10 "-DSTKG_HALF_MINB=10"
cp variants/base.so paper_1912_10082_b200/_stk_gpu.so
touch paper_1912_10082_b200/_stk_gpu.so
