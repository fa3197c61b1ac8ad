cd $GRAFT_REPO_ROOT
./tools/microbench/gemm_bench > gpurun_out/gemm_bench.txt 2>&1; echo rc=$?
cat gpurun_out/gemm_bench.txt
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; echo bench rc=$?; cat gpurun_out/bench.log
