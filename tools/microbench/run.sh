#!/bin/bash
# one-shot GPU probe: FP64 peaks, cuBLAS DGEMM, host facts
mkdir -p gpurun_out
(nproc; lscpu | grep -E "Model name|Socket|Thread|Core"; free -g; nvidia-smi) > gpurun_out/host.txt 2>&1
./tools/microbench/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
python tools/microbench/cublas_dgemm.py > gpurun_out/cublas_dgemm.txt 2>&1
cat gpurun_out/host.txt gpurun_out/fp64_peak.txt gpurun_out/cublas_dgemm.txt
